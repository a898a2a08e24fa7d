/*
 * ORACLE TEST INFRASTRUCTURE — CPU restatement of the reference hot path.
 *
 * Plain C11, complex128, no FMA contraction (built with -ffp-contract=off):
 * a restatement of the reference algorithm (arXiv 2108.05665 `mtc`,
 * /root/reference/proj) that consumes the same POD problem as the product's
 * C ABI (include/mtcg.h). Only tests/, __graft_entry__.smoke() and bench.py's
 * CPU-baseline leg may load it, and only as the checker.
 *
 * Pinning: tests/test_oracle.py checks it against the reference's golden
 * vectors (Fig. 7 amplitudes, node counts, sliced H, batch legs, XEB rows)
 * and bit-for-bit against the reference library itself (oracle/_ref) on
 * random instances — see tests/golden/.
 */
#ifndef MTC_ORACLE_H
#define MTC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/mtcg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes follow mtcg_status. */

/* eval_naive / eval_all / eval_sliced semantics (multieval.cpp:384-516):
 * mode is an mtcg_eval_mode. out_values: n_requests * 2^w complex (re, im).
 * node_contractions: [n_nodes] or NULL. counters: {mults, adds, rw}. */
int orc_eval(const mtcg_problem* p, int mode, double* out_values,
             uint64_t values_capacity, uint64_t* node_contractions,
             uint64_t* counters, int32_t* out_legs, int32_t* n_out_legs,
             char* err, size_t errlen);

/* Same, folding only slices [s_begin, min(s_end, S)) (a rank's partial). */
int orc_eval_slices(const mtcg_problem* p, int mode, uint64_t s_begin,
                    uint64_t s_end, double* out_values,
                    uint64_t values_capacity, uint64_t* node_contractions,
                    uint64_t* counters, int32_t* out_legs, int32_t* n_out_legs,
                    char* err, size_t errlen);

/* One pairwise contraction with the reference kernel's exact reduction
 * order (contract_pair, tensor.cpp:150-253). Legs are ids; dims all given.
 * out_legs receives the result legs (ascending); returns their count or -1
 * on a data error. */
int orc_contract_pair(int ra, const uint32_t* a_legs, const uint32_t* a_dims,
                      const double* a, int rb, const uint32_t* b_legs,
                      const uint32_t* b_dims, const double* b, int nclosed,
                      const uint32_t* closed, uint32_t* out_legs,
                      uint32_t* out_dims, double* out, uint64_t* counters);

/* linear_xeb (xeb.cpp:28-50) with the Neumaier compensated sum. */
int orc_linear_xeb(int n, const double* probs, uint64_t count, double* out,
                   char* err, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif
