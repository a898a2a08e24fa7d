// Paper-scale request ingestion: the reference's sample
// reader (read_samples, formats.cpp:42-69), the per-slot ranking of
// build_assignments (diagram.cpp:229-297) and the amplitude TSV rows with '*'
// expansion (format_amplitude_row formats.cpp:78-83, tools/main.cpp:161-179),
// natively and split over host threads by row ranges — at 10^6 requests the
// reference's one-line-at-a-time string handling is the serial prefix of a
// run. Host code: the work is byte parsing and table lookups whose output
// (the n x slots tuple matrix) the host planner consumes, so a device pass
// would only add two PCIe copies of it. Same results and error messages as
// the reference (ParseError "line N: ...", DataError).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ingest.hpp"
#include "planner.hpp"

namespace mtcg {

namespace {

unsigned n_threads(uint64_t work) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  return work >= (uint64_t{1} << 20) ? hw : 1u;
}

template <class F>
void parallel(unsigned nt, F&& f) {
  if (nt <= 1) {
    f(0u);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nt);
  for (unsigned t = 0; t < nt; ++t) th.emplace_back([&f, t] { f(t); });
  for (auto& x : th) x.join();
}

struct LineError {
  uint64_t line = ~uint64_t{0};
  std::string msg;
};

}  // namespace

// ---- read_samples (formats.cpp:42-69) --------------------------------------------

SampleMatrix read_samples(const char* text, uint64_t len, int bit_order) {
  // chunks start after a newline so every chunk holds whole lines
  const unsigned nt = n_threads(len);
  std::vector<uint64_t> start(nt + 1, len);
  start[0] = 0;
  for (unsigned t = 1; t < nt; ++t) {
    uint64_t p = std::max(start[t - 1], len * t / nt);
    const void* nl = p < len ? std::memchr(text + p, '\n', len - p) : nullptr;
    start[t] = nl ? static_cast<uint64_t>(static_cast<const char*>(nl) - text) + 1 : len;
  }
  // line numbers: newlines before each chunk
  std::vector<uint64_t> nl_count(nt, 0);
  parallel(nt, [&](unsigned t) {
    uint64_t c = 0;
    for (uint64_t p = start[t]; p < start[t + 1]; ++p) c += text[p] == '\n';
    nl_count[t] = c;
  });
  struct Chunk {
    std::string rows;       // canonical rows back to back
    uint64_t n = 0;
    int width = -1;         // first row's width
    uint64_t first_line = 0;
    LineError err;          // first character / internal length error
  };
  std::vector<Chunk> ch(nt);
  parallel(nt, [&](unsigned t) {
    Chunk& c = ch[t];
    uint64_t line = 1;
    for (unsigned u = 0; u < t; ++u) line += nl_count[u];
    uint64_t p = start[t];
    const uint64_t end = start[t + 1];
    while (p < end) {
      const char* nl = static_cast<const char*>(std::memchr(text + p, '\n', end - p));
      uint64_t e = nl ? static_cast<uint64_t>(nl - text) : end;
      const uint64_t next = nl ? e + 1 : end;
      // '#' comment, then trim " \t\r" (formats.cpp:28-33)
      const void* hash = std::memchr(text + p, '#', e - p);
      if (hash) e = static_cast<uint64_t>(static_cast<const char*>(hash) - text);
      uint64_t b = p;
      while (b < e && (text[b] == ' ' || text[b] == '\t' || text[b] == '\r')) ++b;
      while (e > b && (text[e - 1] == ' ' || text[e - 1] == '\t' || text[e - 1] == '\r')) --e;
      if (e > b) {
        for (uint64_t q = b; q < e; ++q) {
          const char x = text[q];
          if (x != '0' && x != '1' && x != '*') {
            c.err = {line, std::string("invalid bitstring character '") + x + "'"};
            return;
          }
        }
        const int w = static_cast<int>(e - b);
        if (c.width < 0) {
          c.width = w;
          c.first_line = line;
        } else if (w != c.width) {
          c.err = {line, "bitstring length differs from previous lines"};
          return;
        }
        if (bit_order == 1) {
          for (uint64_t q = e; q-- > b;) c.rows.push_back(text[q]);
        } else {
          c.rows.append(text + b, e - b);
        }
        ++c.n;
      }
      ++line;
      p = next;
    }
  });
  // the earliest error in line order: a chunk's own error, or its first row
  // disagreeing in length with the first row of the whole file
  LineError first;
  int width = -1;
  for (unsigned t = 0; t < nt; ++t) {
    const Chunk& c = ch[t];
    if (c.width >= 0) {
      if (width < 0) {
        width = c.width;
      } else if (c.width != width) {
        if (c.first_line < first.line) first = {c.first_line, "bitstring length differs from previous lines"};
        break;  // later chunks only hold later lines
      }
    }
    if (c.err.line < first.line) first = c.err;
    if (c.err.line != ~uint64_t{0}) break;
  }
  if (first.line != ~uint64_t{0}) throw ParseError(first.msg, first.line);
  SampleMatrix m;
  m.n_qubits = width < 0 ? 0 : width;
  for (const Chunk& c : ch) m.n_rows += c.n;
  m.chars.reserve(m.n_rows * static_cast<uint64_t>(std::max(width, 0)));
  for (const Chunk& c : ch) m.chars.append(c.rows);
  // one '*' pattern (formats.cpp:61-67)
  if (m.n_rows > 1) {
    const int nq = m.n_qubits;
    const char* f = m.chars.data();
    const unsigned T = n_threads(m.chars.size());
    std::vector<char> bad(T, 0);
    parallel(T, [&](unsigned t) {
      const uint64_t i0 = 1 + (m.n_rows - 1) * t / T, i1 = 1 + (m.n_rows - 1) * (t + 1) / T;
      for (uint64_t i = i0; i < i1 && !bad[t]; ++i)
        for (int q = 0; q < nq; ++q)
          if ((f[i * nq + q] == '*') != (f[q] == '*')) {
            bad[t] = 1;
            break;
          }
    });
    for (char b : bad)
      if (b) throw ParseError("'*' positions differ between sample lines", 0);
  }
  return m;
}

// ---- build_assignments' per-slot ranking (diagram.cpp:229-297) ------------------

Assignment assign(const char* s, uint64_t n, int nq, int n_slots, const int32_t* slot_qubit_begin,
                  const int32_t* slot_qubits, uint32_t* tuples) {
  Assignment a;
  // batch positions: the '*' columns of the first sample (tools/main.cpp
  // batch_legs_of); every sample must agree (diagram.cpp:249-258)
  std::vector<char> is_batch(nq, 0);
  if (n)
    for (int q = 0; q < nq; ++q) is_batch[q] = s[q] == '*';
  {
    const unsigned nt = n_threads(n * static_cast<uint64_t>(nq));
    std::vector<uint64_t> bad(nt, ~uint64_t{0});
    parallel(nt, [&](unsigned t) {
      for (uint64_t i = n * t / nt; i < n * (t + 1) / nt; ++i)
        for (int q = 0; q < nq; ++q) {
          const char x = s[i * nq + q];
          if ((x != '0' && x != '1' && x != '*') || (x == '*') != static_cast<bool>(is_batch[q])) {
            bad[t] = i * nq + q;
            return;
          }
        }
    });
    for (uint64_t b : bad)
      if (b != ~uint64_t{0}) {
        const uint64_t i = b / nq;
        const int q = static_cast<int>(b % nq);
        const std::string row(s + i * nq, nq);
        const char x = s[b];
        if (x != '0' && x != '1' && x != '*')
          throw DataError("bitstring '" + row + "' has invalid character '" + std::string(1, x) + "'");
        throw DataError("bitstring '" + row + "' position " + std::to_string(q) +
                        (x == '*' ? " is '*' but not a batch position" : " must be '*' (batch position)"));
      }
  }
  for (int j = 0; j < n_slots; ++j)
    for (int x = slot_qubit_begin[j]; x < slot_qubit_begin[j + 1]; ++x)
      if (slot_qubits[x] < 0 || slot_qubits[x] >= nq) throw DataError("slot qubit index out of range");
  // fixed (non-batch) qubits per slot, slot_open_legs order
  std::vector<std::vector<int>> fixed(n_slots);
  for (int j = 0; j < n_slots; ++j)
    for (int x = slot_qubit_begin[j]; x < slot_qubit_begin[j + 1]; ++x)
      if (!is_batch[slot_qubits[x]]) fixed[j].push_back(slot_qubits[x]);
  for (int j = 0; j < n_slots; ++j)
    if (fixed[j].size() > 24) throw DataError("more than 24 fixed output bits on one slot");
  // key of row i on slot j: the fixed bits, first fixed qubit most
  // significant (ascending keys = the reference's ascending bit tuples);
  // flattened so the per-row loops touch two small arrays
  std::vector<int32_t> fb(n_slots + 1, 0), fq;
  for (int j = 0; j < n_slots; ++j) {
    fq.insert(fq.end(), fixed[j].begin(), fixed[j].end());
    fb[j + 1] = static_cast<int32_t>(fq.size());
  }
  fq.push_back(0);
  const int32_t* FB = fb.data();
  const int32_t* FQ = fq.data();
  auto key = [&](const char* r, int j) {
    uint32_t k = 0;
    for (int x = FB[j]; x < FB[j + 1]; ++x) k = (k << 1) | static_cast<uint32_t>(r[FQ[x]] == '1');
    return k;
  };
  // pass 1: present keys per slot (per-thread presence tables, merged)
  std::vector<uint64_t> off(n_slots + 1, 0);
  for (int j = 0; j < n_slots; ++j) off[j + 1] = off[j] + (uint64_t{1} << fixed[j].size());
  const unsigned nt = n_threads(n * static_cast<uint64_t>(n_slots));
  std::vector<std::vector<uint8_t>> seen(nt, std::vector<uint8_t>(off[n_slots], 0));
  std::vector<int> live;  // slots with fixed bits
  for (int j = 0; j < n_slots; ++j)
    if (!fixed[j].empty()) live.push_back(j);
  parallel(nt, [&](unsigned t) {
    uint8_t* sn = seen[t].data();
    for (uint64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) {
      const char* r = s + i * nq;
      for (int j : live) sn[off[j] + key(r, j)] = 1;
    }
  });
  for (unsigned t = 1; t < nt; ++t)
    for (uint64_t x = 0; x < off[n_slots]; ++x) seen[0][x] |= seen[t][x];
  // ranks: distinct keys ascending (std::map order in the reference)
  std::vector<uint32_t> rank(off[n_slots], 0);
  a.slot_n_values.assign(n_slots, 1);
  a.value_key_begin.assign(n_slots + 1, 0);
  for (int j = 0; j < n_slots; ++j) {
    if (fixed[j].empty() || n == 0) {
      a.value_keys.push_back(0);  // the slot tensor itself
    } else {
      uint32_t v = 0;
      for (uint64_t k = 0; k < (uint64_t{1} << fixed[j].size()); ++k)
        if (seen[0][off[j] + k]) {
          rank[off[j] + k] = v++;
          a.value_keys.push_back(static_cast<uint32_t>(k));
        }
      a.slot_n_values[j] = static_cast<int32_t>(v);
    }
    a.value_key_begin[j + 1] = a.value_keys.size();
    a.fixed_bits.push_back(static_cast<int32_t>(fixed[j].size()));
  }
  // pass 2: the tuple matrix, written in place (row-major, whole rows)
  if (tuples)
    parallel(nt, [&](unsigned t) {
      for (uint64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) {
        const char* r = s + i * nq;
        uint32_t* row = tuples + i * n_slots;
        for (int j = 0; j < n_slots; ++j) row[j] = FB[j] == FB[j + 1] ? 0u : rank[off[j] + key(r, j)];
      }
    });
  return a;
}

// ---- amplitude TSV rows (formats.cpp:78-83, tools/main.cpp:161-179) ----------------

std::string format_amplitudes(const char* s, uint64_t n, int nq, int bit_order, const double* values, int w) {
  std::vector<int> stars;
  if (n)
    for (int q = 0; q < nq; ++q)
      if (s[q] == '*') stars.push_back(q);
  if (static_cast<int>(stars.size()) != w)
    throw DataError("value tensors have " + std::to_string(w) + " batch legs, samples have " +
                    std::to_string(stars.size()) + " '*' positions");
  const uint64_t per = uint64_t{1} << w;
  const unsigned nt = n_threads(n * per * 48);
  std::vector<std::string> part(nt);
  parallel(nt, [&](unsigned t) {
    std::string& o = part[t];
    std::string bits(nq, '0');
    char buf[96];
    for (uint64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) {
      for (uint64_t v = 0; v < per; ++v) {
        std::memcpy(&bits[0], s + i * nq, nq);
        // '*' positions in row-major order of the batch legs (ascending
        // qubit): the last position is the least significant bit of v
        uint64_t rest = v;
        for (size_t x = stars.size(); x-- > 0;) {
          bits[stars[x]] = (rest & 1) ? '1' : '0';
          rest >>= 1;
        }
        if (bit_order == 1) {
          for (int q = nq; q-- > 0;) o.push_back(bits[q]);
        } else {
          o.append(bits);
        }
        const double* a = values + 2 * (i * per + v);
        const int len = std::snprintf(buf, sizeof buf, "\t%.16e\t%.16e\n", a[0], a[1]);
        o.append(buf, len);
      }
    }
  });
  std::string out;
  size_t total = 0;
  for (auto& p : part) total += p.size();
  out.reserve(total);
  for (auto& p : part) out.append(p);
  return out;
}

}  // namespace mtcg
