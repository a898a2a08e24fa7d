// Paper-scale request ingestion (ingest.cpp): samples text -> canonical
// sample matrix, per-slot value ranking -> tuple matrix, amplitude TSV rows.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace mtcg {

struct SampleMatrix {
  uint64_t n_rows = 0;
  int n_qubits = 0;
  std::string chars;  // [n_rows][n_qubits], canonical (qubit 0 first)
};
// read_samples (formats.cpp:42-69); bit_order 1 = qubit 0 last (reversed)
SampleMatrix read_samples(const char* text, uint64_t len, int bit_order);

struct Assignment {
  std::vector<int32_t> slot_n_values;     // [n_slots]
  std::vector<uint64_t> value_key_begin;  // [n_slots + 1]
  std::vector<uint32_t> value_keys;       // distinct fixed-bit tuples, ascending
  std::vector<int32_t> fixed_bits;        // [n_slots]
};
// build_assignments' ranking (diagram.cpp:229-297) over slot_qubits CSR;
// the tuple matrix [n][n_slots] is written to `tuples` (null: not written)
Assignment assign(const char* samples, uint64_t n, int n_qubits, int n_slots, const int32_t* slot_qubit_begin,
                  const int32_t* slot_qubits, uint32_t* tuples);

// amplitude TSV (format_amplitude_row, formats.cpp:78-83) with '*' expansion
// (tools/main.cpp:161-179); values [n][2^w] complex
std::string format_amplitudes(const char* samples, uint64_t n, int n_qubits, int bit_order, const double* values,
                              int w);

}  // namespace mtcg
