/*
 * TEST INFRASTRUCTURE ONLY — the CPU parity oracle. Never linked into or
 * called by the product (paper_2209_06800_b200/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * load liboracle.so, and only as the checker or the timed CPU baseline.
 *
 * Two halves:
 *
 * 1. Partition metadata restatement (pinned): Alg. 1 split, address
 *    translation, local/remote classification, ps-slicing and the dist
 *    interleave. Written as plain left-to-right scans, independent of the
 *    product's builder, and checked bit-for-bit against the reference library
 *    itself (oracle/_ref/libpipeshard_ref.so) and the reference's own
 *    known-answer tests (tests/test_oracle.py).
 *
 * 2. GCN/GIN layer forward (PARITY UNPINNED by reference code): the reference
 *    (pipeshard) stores no embedding values (R:SPEC.md:121-124) and has no
 *    layer arithmetic, so this is a restatement of the paper's equations —
 *    R:PAPER.md:33-38 (aggregate over N(v) ∪ {v}), 504-508 (2-layer GCN,
 *    Z = softmax(Â ReLU(Â X W1) W2), Â = A + I), 511-517 (GIN,
 *    h' = MLP((1+eps) h_v + Σ_{u∈N(v)} h_u)). It is pinned only by hand
 *    known-answer tests and an fp64-vs-fp32 cross-check (tests/golden/).
 *
 * Graph convention (R:SPEC.md:105-111): directed CSR, row v = target, its
 * columns are the neighbors whose rows are gathered; duplicates and
 * self-loops in the CSR are kept and summed like any other neighbor.
 */
#ifndef MGG_ORACLE_H_
#define MGG_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- metadata restatement ------------------------------------------------ */

/* Alg. 1 as a linear scan (R:proj/src/placement.cpp:44-71,
 * R:proj/tests/test_util.hpp:31-53). out: num_gpus-1 split points. */
void orc_split_points(uint64_t n, const uint64_t* row_ptr, uint32_t num_gpus,
                      uint64_t* out);

/* Placement ranges, 2*num_gpus entries (lb,ub). mode 0 equal_nodes,
 * 1 follow_split (R:proj/src/placement.cpp:73-106). */
void orc_placement(uint64_t n, const uint64_t* row_ptr, uint32_t num_gpus,
                   int mode, uint64_t* ranges);

/* translate (R:proj/src/placement.cpp:108-119) by scanning the ranges. */
void orc_translate(uint32_t num_gpus, const uint64_t* ranges, uint64_t id,
                   uint32_t* gpu, uint64_t* off);

/* Number of ps-partitions of each kind the local/remote split of `gpu` yields
 * (R:proj/src/workload.cpp:26-82) and the edge counts. counts[4] =
 * {local_parts, remote_parts, local_edges, remote_edges}. */
void orc_partition_counts(uint64_t n, const uint64_t* row_ptr,
                          const uint64_t* col, uint32_t num_gpus,
                          const uint64_t* ranges, const uint64_t* chunk,
                          uint32_t gpu, uint32_t ps, uint64_t* counts);

/* Warp tasks of warp w under the interleaved mapping
 * (R:proj/src/workload.cpp:103-124). Writes up to 2*dist (kind,index) pairs
 * into kinds/idx and returns the count. */
uint32_t orc_warp_tasks(uint64_t n_local, uint64_t n_remote, uint32_t dist,
                        uint64_t w, uint8_t* kinds, uint32_t* idx);

/* ---- layer forward (fp64 accumulate unless noted) ------------------------ */

/* out[v] = self_scale * x[v] + Σ_{u ∈ col[row_ptr[v]..row_ptr[v+1])} x[u]
 * for v in [row_lo, row_hi); x row-major n x d. norm: 0 none, 1 sym
 * (D^-1/2 (A+I) D^-1/2 with d_v = row degree + 1). relu_in applies ReLU to
 * every gathered/self row first. acc64 selects double (1) or float (0)
 * accumulation; threads 0 = all. */
void orc_aggregate(int acc64, int threads, uint64_t n, const uint64_t* row_ptr,
                   const uint64_t* col, const float* x, uint32_t d,
                   double self_scale, int norm, int relu_in, uint64_t row_lo,
                   uint64_t row_hi, float* out);

/* y = act(x W + b); x n x k, W k x m row-major; b may be NULL.
 * act: 0 none, 1 relu, 2 row softmax. */
void orc_dense(int acc64, int threads, uint64_t n, const float* x, uint32_t k,
               const float* w, const float* b, uint32_t m, int act, float* y);

/* 2-layer GCN (R:PAPER.md:504-508): logits = Â ReLU(Â X W1) W2,
 * z = softmax(logits). h1 (n x hidden, post-ReLU) and logits (n x classes)
 * may be NULL. */
void orc_gcn2_forward(int acc64, int threads, uint64_t n,
                      const uint64_t* row_ptr, const uint64_t* col,
                      const float* x, uint32_t d, const float* w1,
                      uint32_t hidden, const float* w2, uint32_t classes,
                      int norm, float* h1, float* logits, float* z);

/* L-layer GIN (R:PAPER.md:511-517). Layer l: a = (1+eps) h + Σ h_u;
 * t = ReLU(a W1[l] + b1[l]); o = t W2[l] + b2[l]; h = ReLU(o) for l < L-1,
 * z = softmax(o) for the last layer. dims[0] = input dim, dims[l+1] = output
 * width of layer l; every MLP has hidden width `hidden`. Weights are packed
 * layer after layer in w1 (dims[l] x hidden), b1 (hidden), w2 (hidden x
 * dims[l+1]), b2 (dims[l+1]). logits (n x dims[L]) may be NULL. */
void orc_gin_forward(int acc64, int threads, uint64_t n,
                     const uint64_t* row_ptr, const uint64_t* col,
                     const float* x, uint32_t layers, const uint32_t* dims,
                     uint32_t hidden, const float* w1, const float* b1,
                     const float* w2, const float* b2, double eps,
                     float* logits, float* z);

/* ---- synthetic inputs (bench.py --impl reference builds its graph with
 * these or with oracle/_ref, never with the product) --------------------- */
uint64_t orc_gen_synthetic(int kind, uint64_t n, double avg, uint64_t seed,
                           uint64_t* row_ptr, uint64_t* col);
void orc_gen_rmat(uint64_t n, uint64_t m, uint64_t seed, double a, double b, double c,
                  uint64_t* row_ptr, uint64_t* col);

#ifdef __cplusplus
}
#endif
#endif /* MGG_ORACLE_H_ */
