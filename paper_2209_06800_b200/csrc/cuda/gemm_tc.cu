// K2 — Update GEMM on the 5th-gen tensor cores: out = act(pre(X) · W + b).
//
// tcgen05.mma kind::tf32 with a 3xTF32 split so the product keeps fp32
// accuracy (the 1e-4 parity bar): X = Xh + Xl, W = Wh + Wl with Xh, Wh
// exact TF32 values (low 13 mantissa bits cleared) and
//   X·W ≈ Xh·Wh + Xh·Wl + Xl·Wh        (dropped Xl·Wl term ~ 2^-22 |X||W|).
// The GEMM is HBM-bound at these widths (N <= 64, ~2N flop per X byte), so
// the 3x tensor work is free; what matters is streaming X at HBM rate.
//
// Persistent CTA per SM, warp-specialised:
//   warp 0   : TMA producer — X tiles (128 rows x 32 fp32, 128-B swizzle)
//              into a smem ring; W^T hi/lo (and the chain's W2) resident.
//   warp 1   : MMA issuer — one thread; A operands from TMEM:
//              [Xh·Wh | Xh·Wl] (N = 2NP) + Xl·Wh per K=8 step into a TMEM
//              accumulator ring.
//   warp 2   : TMEM allocator.
//   warps 4-7: split — thread = tile row = TMEM lane: pre-transform, Xh/Xl
//              into TMEM (tcgen05.st), releases the smem stage; in the chain
//              variant also turns the first product into the second GEMM's
//              A operand (O never leaves TMEM).
//   warps 8+ : 1-4 epilogue warpgroups — tcgen05.ld, bias / ReLU / row
//              softmax / scaled accumulator seed, 128-B swizzled staging and
//              TMA bulk tensor stores.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace mgg::dev {
namespace {

constexpr int BM = 128;            // rows per tile (UMMA M)
constexpr int BK = 32;             // fp32 per 128-B swizzle row
constexpr int kTileBytes = BM * BK * 4;  // 16 KB
constexpr uint32_t kMaxStages = 8;
constexpr uint32_t kLoSlots = 2;  // Xl twin tiles (decoupled from the TMA ring)
// EG epilogue warpgroups drain max(EG, 2) TMEM accumulators round-robin:
// four for the short-K heads (epilogue-bound: softmax over a row per thread),
// two while a thread's row of NP fp32 fits the 128-register budget of a
// 512-thread CTA, else one.
template <int EG>
constexpr int kThreadsFor = 256 + 128 * EG;
template <int EG>
constexpr uint32_t kNAcc = EG < 2 ? 2 : EG;

struct TcArgs {
  uint64_t rows;
  uint32_t k, n_kb, m, out_pitch;
  uint32_t pre, act, stages;
  const float* bias;
  const float* pre_bias;
  float* out;
  float* out2;
  float out2_scale;
  const float* bias1;  // CHAIN: bias of the first product (m1 = NP columns)
  uint32_t m1;
  const float* row_scale;  // optional per-row multiplier of the product (before bias)
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                       int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}
// Bulk tensor store smem -> global (the epilogue): 32 rows x 128 B,
// 128-B swizzled, clipped by the tensor map at the tensor edges.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x,
                                             int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
      "r"(su32(src)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// UMMA shared-memory descriptor, K-major, 128-B swizzle: rows of 128 B,
// 8-row core groups 1024 B apart (SBO), LBO unused (1), version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (1ull << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// A operand from TMEM (lanes = rows, 32-bit columns = k): the Xl term.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// 16 consecutive 32-bit TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 16 accumulator columns of this warp's 32 TMEM lanes; no wait (callers
// batch several loads behind one tmem_wait).
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

// TMEM column map (NP = padded output width; accumulators are
// [Xh·Wh + Xl·Wh | Xh·Wl], 2·NP columns, double-buffered):
//   [0, 4NP)                 accumulators 0 and 1
//   kXlCol + BK·l, l < 2     Xl k-block slots   } written by the split
//   kXhCol + BK·l            Xh k-block slots   } warpgroup, read by the MMA
//   kOlCol / kOhCol          CHAIN: the intermediate O = act1(X·W + b1) split
//                            into lo/hi, the A operand of the second GEMM
// Xh and Xl live in TMEM so the MMA reads no X from shared memory (the smem
// stage is released by the split itself); accumulating all three products
// into one NP-wide accumulator instead was measured no faster and loses the
// small terms' low bits (softmax error crossed 1e-4).
template <int NP, bool CHAIN, uint32_t NACC>
struct TmemMap {
  static constexpr uint32_t kAccCols = 2 * NP;
  static constexpr uint32_t kXlCol = NACC * kAccCols;
  static constexpr uint32_t kXhCol = kXlCol + kLoSlots * BK;
  static constexpr uint32_t kOlCol = kXhCol + kLoSlots * BK;  // CHAIN: NP columns each
  static constexpr uint32_t kOhCol = kOlCol + NP;
  static constexpr uint32_t kCols = CHAIN ? kOhCol + NP : kOlCol;
  static constexpr uint32_t kAlloc = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128
                                     : kCols <= 256 ? 256 : 512;
  static_assert(kCols <= 512, "TMEM holds 512 columns");
};

// Epilogue staging per warp: NB column blocks of 32 rows x 128 B (one TMA
// store box each), 128-B swizzled so the row-per-lane float4 writes are
// bank-conflict free.
template <int NP>
constexpr int kStoreBlocks = (NP + 31) / 32;
template <int NP, int EG>
constexpr uint32_t kEpBytes = EG * 4 * kStoreBlocks<NP> * 4096;

// out = act(pre(X)·W + b) [+ out2 = out2_scale·(pre(X)·W + b)]; with CHAIN
// the product goes through a second GEMM first:
//   O = ReLU(pre(X)·W + b1)          (kept in TMEM, never written)
//   out = O·W2 (+ out2 = out2_scale·O·W2)
// — the GIN layer boundary Linear2 -> ReLU -> next layer's Linear1 + seed.
template <int NP, bool CHAIN, int EG>
__global__ void __launch_bounds__(kThreadsFor<EG>, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_x,
                   const __grid_constant__ CUtensorMap map_w,
                   const __grid_constant__ CUtensorMap map_w2,
                   const __grid_constant__ CUtensorMap map_out,
                   const __grid_constant__ CUtensorMap map_out2, TcArgs a) {
  static_assert(!CHAIN || EG <= 2, "the chain reuses accumulators j & 1");
  constexpr uint32_t NACC = kNAcc<EG>;
  using TM = TmemMap<NP, CHAIN, NACC>;
  constexpr uint32_t kAccCols = TM::kAccCols;
  constexpr uint32_t kIdescBase = (1u << 4) | (2u << 7) | (2u << 10) | ((BM >> 4) << 24);
  constexpr uint32_t kIdesc2 = kIdescBase | (static_cast<uint32_t>((2 * NP) >> 3) << 17);
  constexpr uint32_t kIdesc1 = kIdescBase | (static_cast<uint32_t>(NP >> 3) << 17);
  constexpr uint32_t kW2Bytes = CHAIN ? (NP / BK) * 2 * NP * 128 : 0;  // W2: K = NP
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the 128-B swizzle, by offsetting the shared array
  // itself (a round trip through uintptr_t would lose the address space and
  // turn every staging access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  const uint32_t wbytes = a.n_kb * 2 * NP * 128;
  uint8_t* w_s = smem;                          // [kb][hi|lo][NP][128 B]
  uint8_t* w2_s = smem + wbytes;                // CHAIN: [NP/BK][hi|lo][NP][128 B]
  uint8_t* x_s = w2_s + kW2Bytes;               // [stage][16 KB] raw X
  uint8_t* ep_s = x_s + a.stages * kTileBytes;  // [groups][4 warps][NB][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ep_s + kEpBytes<NP, EG>);
  uint64_t* full = bars;                        // [stages] TMA -> split
  uint64_t* split = bars + a.stages;            // [stages] split -> MMA (X slots filled)
  uint64_t* empty = bars + 2 * a.stages;        // [stages] split -> TMA
  uint64_t* tfull = bars + 3 * a.stages;        // [NACC] final accumulator -> epilogue
  uint64_t* tempty = tfull + NACC;              // [NACC] epilogue -> MMA
  uint64_t* lofree = tempty + NACC;             // [kLoSlots] MMA -> split (X slots)
  uint64_t* wfull = lofree + kLoSlots;          // W (and W2) resident
  uint64_t* t1full = wfull + 1;                 // CHAIN [2]: first product -> split
  uint64_t* ofull = t1full + 2;                 // CHAIN: O slots filled -> MMA
  uint64_t* ofree = ofull + 1;                  // CHAIN: O slots consumed -> split
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ofree + 1);
  // bias (NP) and pre-bias (n_kb*BK) staged once: the epilogue and split read
  // them as shared-memory broadcasts instead of per-element global loads
  uint8_t* tail = reinterpret_cast<uint8_t*>(ofree + 2);
  float* bias_s = reinterpret_cast<float*>(tail + ((16u - (su32(tail) & 15u)) & 15u));
  float* pb_s = bias_s + NP;
  float* b1_s = pb_s + a.n_kb * BK;  // CHAIN: bias of the first product
  for (uint32_t i = threadIdx.x; i < NP; i += blockDim.x) {
    bias_s[i] = (a.bias && i < a.m) ? __ldg(a.bias + i) : 0.f;
    if (CHAIN) b1_s[i] = (a.bias1 && i < a.m1) ? __ldg(a.bias1 + i) : 0.f;
  }
  if (a.pre == 2)
    for (uint32_t i = threadIdx.x; i < a.n_kb * BK; i += blockDim.x)
      pb_s[i] = i < a.k ? __ldg(a.pre_bias + i) : 0.f;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_tiles = static_cast<uint32_t>((a.rows + BM - 1) / BM);

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 128);
      mbar_init(&empty[s], 128);
    }
    for (uint32_t i = 0; i < NACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 128);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&t1full[i], 1);
    for (uint32_t i = 0; i < kLoSlots; ++i) mbar_init(&lofree[i], 1);
    mbar_init(wfull, 1);
    mbar_init(ofull, 128);
    mbar_init(ofree, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(TM::kAlloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
      mbar_expect_tx(wfull, wbytes + kW2Bytes);
      for (uint32_t kb = 0; kb < a.n_kb; ++kb) {
        tma_2d(w_s + kb * 2 * NP * 128, &map_w, wfull, kb * BK, 0);
        tma_2d(w_s + kb * 2 * NP * 128 + NP * 128, &map_w, wfull, kb * BK, NP);
      }
      if constexpr (CHAIN)
        for (uint32_t kb = 0; kb < static_cast<uint32_t>(NP / BK); ++kb) {
          tma_2d(w2_s + kb * 2 * NP * 128, &map_w2, wfull, kb * BK, 0);
          tma_2d(w2_s + kb * 2 * NP * 128 + NP * 128, &map_w2, wfull, kb * BK, NP);
        }
      uint32_t s = 0, ph = 0;
      for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x)
        for (uint32_t kb = 0; kb < a.n_kb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], kTileBytes);
          tma_2d(x_s + s * kTileBytes, &map_x, &full[s], kb * BK, t * BM);
          if (++s == a.stages) s = 0, ph ^= 1;
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      mbar_wait(wfull, 0);
      uint32_t s = 0, ph = 0, kcount = 0;
      // [Ah·Wh | Ah·Wl] + Al·Wh over `nk` k-blocks whose A slots are TMEM
      // columns al/ah + BK·kb
      auto gemm = [&](uint32_t d, uint32_t al, uint32_t ah, const uint8_t* wsm, uint32_t kb,
                      bool first) {
        const uint64_t wh = umma_desc(su32(wsm + kb * 2 * NP * 128));  // [Wh; Wl]
#pragma unroll
        for (uint32_t k = 0; k < BK / 8; ++k) {  // K=8 per tf32 MMA: +32 B / +8 cols
          const uint64_t o = 2 * k;
          mma_tf32_ts(d, ah + 8 * k, wh + o, kIdesc2, !(first && k == 0));  // [Ah·Wh | Ah·Wl]
          mma_tf32_ts(d, al + 8 * k, wh + o, kIdesc1, 1);                   // += Al·Wh
        }
      };
      // CHAIN: the second product of tile j reuses tile j's accumulator once
      // the split warpgroup has turned it into O
      auto second = [&](uint32_t j) {
        const uint32_t acc = j & 1;
        mbar_wait(ofull, j & 1);
        tc_fence_after();
        if constexpr (CHAIN)
          for (uint32_t kb = 0; kb < static_cast<uint32_t>(NP / BK); ++kb)
            gemm(tmem + acc * kAccCols, tmem + TM::kOlCol + BK * kb,
                 tmem + TM::kOhCol + BK * kb, w2_s, kb, kb == 0);
        mma_commit(ofree);
        mma_commit(&tfull[acc]);
      };
      uint32_t it = 0;
      for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        const uint32_t acc = it % NACC, aph = (it / NACC) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * kAccCols;
        for (uint32_t kb = 0; kb < a.n_kb; ++kb, ++kcount) {
          const uint32_t l = kcount % kLoSlots;
          mbar_wait(&split[s], ph);
          tc_fence_after();
          gemm(d, tmem + TM::kXlCol + BK * l, tmem + TM::kXhCol + BK * l, w_s, kb, kb == 0);
          mma_commit(&lofree[l]);  // X slot l free once these MMAs retire
          if (++s == a.stages) s = 0, ph ^= 1;
        }
        if (CHAIN) {
          mma_commit(&t1full[acc]);
          if (it > 0) second(it - 1);
        } else {
          mma_commit(&tfull[acc]);
        }
      }
      if (CHAIN && it > 0) second(it - 1);
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- split warpgroup: thread = tile row = TMEM lane
    const int row = threadIdx.x - 128;  // 0..127
    const uint32_t lane_base = static_cast<uint32_t>(32 * (warp % 4)) << 16;
    uint32_t s = 0, ph = 0, kcount = 0;
    // 16 values -> TMEM Xh/Xl style slots (hi = TF32-truncated, lo = rest);
    // the stores complete (wait::st) before the caller signals the MMA
    auto split_store = [&](float* v, uint32_t lo_col, uint32_t hi_col) {
      float lov[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float h = tf32_hi(v[q]);
        lov[q] = v[q] - h;
        v[q] = h;
      }
      tmem_st16(tmem + lo_col + lane_base, lov);
      tmem_st16(tmem + hi_col + lane_base, v);
    };
    auto st_wait = [] { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); };
    // CHAIN: O(j) = ReLU(first product + b1) from accumulator j&1 into the O slots
    auto make_o = [&](uint32_t j) {
      const uint32_t acc = j & 1;
      mbar_wait(&t1full[acc], (j >> 1) & 1);
      if (j > 0) mbar_wait(ofree, (j - 1) & 1);  // O(j-1) consumed by the second GEMM
      tc_fence_after();
      const uint32_t ta = tmem + acc * kAccCols + lane_base;
#pragma unroll
      for (int c0 = 0; c0 < NP; c0 += 16) {
        uint32_t h[16], l[16];
        tmem_ld16_nowait(ta + c0, h);
        tmem_ld16_nowait(ta + NP + c0, l);
        tmem_wait();
        float v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          v[q] = fmaxf(__uint_as_float(h[q]) + __uint_as_float(l[q]) + b1_s[c0 + q], 0.f);
        split_store(v, TM::kOlCol + c0, TM::kOhCol + c0);
      }
      st_wait();
      tc_fence_before();
      mbar_arrive(ofull);
    };
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      for (uint32_t kb = 0; kb < a.n_kb; ++kb, ++kcount) {
        const uint32_t l = kcount % kLoSlots;
        mbar_wait(&full[s], ph);
        mbar_wait(&lofree[l], ((kcount / kLoSlots) & 1) ^ 1);
        const float4* xt = reinterpret_cast<const float4*>(x_s + s * kTileBytes);
#pragma unroll
        for (int half = 0; half < 2; ++half) {  // 16 columns at a time
          float v[16];
#pragma unroll
          for (int c = 0; c < 4; ++c) {  // this row's (swizzled) float4 chunks
            const int cc = half * 4 + c;
            float4 x4 = xt[row * 8 + (cc ^ (row & 7))];
            float* e = &x4.x;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float x = e[q];
              if (a.pre == 2) x += pb_s[kb * BK + cc * 4 + q];
              if (a.pre) x = fmaxf(x, 0.f);
              v[c * 4 + q] = x;
            }
          }
          split_store(v, TM::kXlCol + BK * l + 16 * half, TM::kXhCol + BK * l + 16 * half);
        }
        mbar_arrive(&empty[s]);  // smem stage consumed: back to the TMA
        st_wait();
        tc_fence_before();
        mbar_arrive(&split[s]);
        if (++s == a.stages) s = 0, ph ^= 1;
      }
      if (CHAIN && it > 0) make_o(it - 1);
    }
    if (CHAIN && it > 0) make_o(it - 1);
  } else if (warp >= 8) {
    // ---------------- epilogue warpgroup(s) (overlap the next tiles' split);
    // with two groups, group e drains accumulator e (tiles it % 2 == e)
    const int eg = (warp - 8) / 4;
    const int g = warp % 4;  // TMEM lane quarter
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      if (EG > 1 && static_cast<int>(it % EG) != eg) continue;
      const uint32_t acc = it % NACC, aph = (it / NACC) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      float y[NP];
      const uint32_t ta = tmem + acc * kAccCols + (static_cast<uint32_t>(32 * g) << 16);
      if (EG >= 3) {  // register-lean: 16 columns in flight
#pragma unroll
        for (int c = 0; c < NP; c += 16) {
          uint32_t r[16];
          tmem_ld16_nowait(ta + c, r);
          tmem_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) y[c + q] = __uint_as_float(r[q]);
          tmem_ld16_nowait(ta + NP + c, r);
          tmem_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) y[c + q] += __uint_as_float(r[q]);
        }
      } else {
        uint32_t r[NP];
#pragma unroll
        for (int c = 0; c < NP; c += 16) tmem_ld16_nowait(ta + c, r + c);
        tmem_wait();
#pragma unroll
        for (int c = 0; c < NP; ++c) y[c] = __uint_as_float(r[c]);
#pragma unroll
        for (int c = 0; c < NP; c += 16) tmem_ld16_nowait(ta + NP + c, r + c);
        tmem_wait();
#pragma unroll
        for (int c = 0; c < NP; ++c) y[c] += __uint_as_float(r[c]);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (a.row_scale) {  // normalised GCN: this row's D^-1/2 power
        const uint64_t r = static_cast<uint64_t>(t) * BM + 32 * g + lane;
        const float rs = r < a.rows ? __ldg(a.row_scale + r) : 1.f;
#pragma unroll
        for (int c = 0; c < NP; ++c) y[c] *= rs;
      }
      // Each thread holds its row: write it into the warp's swizzled staging
      // blocks, then one lane hands the 32 x NP tile to the TMA engine (bulk
      // tensor store, clipped at the last row / the pitch) — no per-lane
      // global stores, no smem read-back by the warp.
      uint8_t* ep = ep_s + ((eg * 4 + g) * kStoreBlocks<NP>) * 4096;
      const int row0 = static_cast<int>(t * BM + 32 * g);
      auto stage_and_store = [&](const CUtensorMap* map, float scale) {
        if (lane == 0) bulk_wait_read0();  // the previous store has left the staging
        __syncwarp();
        // columns >= m are exact zeros (W^T and bias zero-padded, softmax
        // zeroes them), so they are staged as they are, no per-column select
        if (scale == 1.f) {
#pragma unroll
          for (int c = 0; c < NP; c += 4) {
            const int b = c / 32, c4 = (c % 32) / 4;
            *reinterpret_cast<float4*>(ep + b * 4096 + lane * 128 + ((c4 ^ (lane & 7)) << 4)) =
                make_float4(y[c], y[c + 1], y[c + 2], y[c + 3]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < NP; c += 4) {
            const int b = c / 32, c4 = (c % 32) / 4;
            *reinterpret_cast<float4*>(ep + b * 4096 + lane * 128 + ((c4 ^ (lane & 7)) << 4)) =
                make_float4(y[c] * scale, y[c + 1] * scale, y[c + 2] * scale, y[c + 3] * scale);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int b = 0; b < kStoreBlocks<NP>; ++b) tma_store_2d(map, ep + b * 4096, 32 * b, row0);
          bulk_commit();
        }
      };
      if (a.bias) {
#pragma unroll
        for (int c = 0; c < NP; c += 4) {
          const float4 b4 = *reinterpret_cast<const float4*>(bias_s + c);
          y[c] += b4.x;
          y[c + 1] += b4.y;
          y[c + 2] += b4.z;
          y[c + 3] += b4.w;
        }
      }
      if (a.out2) stage_and_store(&map_out2, a.out2_scale);
      float oscale = 1.f;  // softmax: 1/sum, applied while staging
      if (a.act == 1) {
#pragma unroll
        for (int c = 0; c < NP; ++c) y[c] = fmaxf(y[c], 0.f);
      } else if (a.act == 2) {
        // NP = round16(m): only the last 16 columns can be padding, so the
        // column test is compile-time true elsewhere
        const int m = static_cast<int>(a.m);
        float mx = -FLT_MAX;
#pragma unroll
        for (int c = 0; c < NP; ++c)
          if (c < NP - 16 || c < m) mx = fmaxf(mx, y[c]);
        // e^(y - mx) = 2^(y·log2e - mx·log2e): one FFMA + MUFU.EX2 per column
        const float l2e = 1.4426950408889634f, off = -mx * l2e;
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < NP; ++c) {
          y[c] = (c < NP - 16 || c < m) ? ex2_approx(fmaf(y[c], l2e, off)) : 0.f;
          sum += y[c];
        }
        oscale = 1.f / sum;
      }
      stage_and_store(&map_out, oscale);
    }
    if (lane == 0) bulk_wait0();  // stores complete before the CTA's smem goes away
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TM::kAlloc));
  }
}

// W (k x m row-major) -> W^T split [hi rows 0..NP) | lo rows NP..2NP), K padded.
__global__ void prep_w_kernel(const float* __restrict__ w, uint32_t k, uint32_t m, uint32_t np,
                              uint32_t kpad, float* __restrict__ out) {
  const uint32_t total = np * kpad;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t n = i / kpad, kk = i % kpad;
    const float x = (n < m && kk < k) ? w[static_cast<size_t>(kk) * m + n] : 0.f;
    const float h = tf32_hi(x);
    out[static_cast<size_t>(n) * kpad + kk] = h;
    out[static_cast<size_t>(np + n) * kpad + kk] = x - h;
  }
}

PFN_cuTensorMapEncodeTiled encode_fn() {
  static PFN_cuTensorMapEncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  });
  if (!fn) throw Status{MGG_E_CUDA, "cuTensorMapEncodeTiled unavailable"};
  return fn;
}

CUtensorMap make_map(const float* base, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
                     uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {pitch_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                 const_cast<float*>(base), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Status{MGG_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")"};
  return m;
}

template <int NP, bool CHAIN, int EG>
void run_tc(const float* in, uint32_t in_pitch, const float* wt, uint32_t kpad,
            const float* wt2, const TcArgs& a, cudaStream_t st) {
  const size_t wbytes = static_cast<size_t>(a.n_kb) * 2 * NP * 128;
  const size_t w2bytes = CHAIN ? static_cast<size_t>(NP / BK) * 2 * NP * 128 : 0;
  TcArgs b = a;
  b.stages = kMaxStages;
  auto smem_for = [&](uint32_t stages) {
    return 1024 + wbytes + w2bytes + stages * kTileBytes + kEpBytes<NP, EG> +
           (3 * stages + 2 * kNAcc<EG> + 7 + kLoSlots) * 8 + 16 + 16 + 4 * (2 * NP + a.n_kb * BK);
  };
  static const uint32_t cap_env = [] {
    const char* e = std::getenv("MGG_TC_STAGES");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
  }();
  if (cap_env) b.stages = std::min<uint32_t>(cap_env, kMaxStages);
  while (b.stages > 2 && smem_for(b.stages) > 227 * 1024) --b.stages;
  if (!cap_env && b.stages > 2 * a.n_kb + 2) b.stages = 2 * a.n_kb + 2;  // no use beyond ~2 tiles
  const size_t smem = smem_for(b.stages);
  if (smem > 227 * 1024) throw Status{MGG_E_CONFIG, "gemm_tc: W too large for smem"};
  const CUtensorMap mx = make_map(in, a.k, a.rows, size_t(in_pitch) * 4, BK, BM);
  const CUtensorMap mw = make_map(wt, kpad, 2 * NP, size_t(kpad) * 4, BK, NP);
  const CUtensorMap mw2 = CHAIN ? make_map(wt2, NP, 2 * NP, size_t(NP) * 4, BK, NP) : mw;
  const CUtensorMap mo = make_map(a.out, a.out_pitch, a.rows, size_t(a.out_pitch) * 4, 32, 32);
  const CUtensorMap mo2 = a.out2 ? make_map(a.out2, a.out_pitch, a.rows,
                                            size_t(a.out_pitch) * 4, 32, 32)
                                 : mo;
  MGG_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<NP, CHAIN, EG>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  int dev = 0, sms = 0;
  MGG_CUDA(cudaGetDevice(&dev));
  MGG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint64_t tiles = (a.rows + BM - 1) / BM;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(tiles, sms));
  gemm_tc_kernel<NP, CHAIN, EG><<<grid, kThreadsFor<EG>, smem, st>>>(mx, mw, mw2, mo, mo2, b);
  MGG_CUDA(cudaGetLastError());
}

}  // namespace

bool gemm_tc_supported(uint32_t k, uint32_t m) {
  static const uint32_t min_k = [] {
    const char* e = std::getenv("MGG_TC_MINK");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 8u;
  }();
  if (m == 0 || m > 64 || k < min_k || k < 8) return false;
  const uint32_t np = (m + 15) / 16 * 16;
  const size_t wbytes = size_t((k + BK - 1) / BK) * 2 * np * 128;
  const size_t kpad = size_t((k + BK - 1) / BK) * BK;
  const size_t ep = size_t(np <= 48 ? 4 : 1) * 4 * ((np + 31) / 32) * 4096;
  return 1024 + wbytes + 2 * kTileBytes + ep + 160 + 16 + 4 * (2 * np + kpad) <= 227 * 1024;
}

// Returns the cached device W^T hi/lo block for `w`, building it on first use.
const float* gemm_tc_prepare(mgg_dbuf* w, uint32_t k, uint32_t m, cudaStream_t st) {
  const uint32_t np = (m + 15) / 16 * 16, kpad = (k + BK - 1) / BK * BK;
  if (!w->tc_cache || w->tc_k != k || w->tc_m != m) {
    if (w->tc_cache) MGG_CUDA(cudaFree(w->tc_cache));
    w->tc_cache = nullptr;
    MGG_CUDA(cudaMalloc(&w->tc_cache, size_t(2) * np * kpad * sizeof(float)));
    prep_w_kernel<<<64, 256, 0, st>>>(static_cast<const float*>(w->ptr), k, m, np, kpad,
                                      static_cast<float*>(w->tc_cache));
    MGG_CUDA(cudaGetLastError());
    w->tc_k = k;
    w->tc_m = m;
  }
  return static_cast<const float*>(w->tc_cache);
}

void launch_dense_tc(const float* in, uint32_t in_pitch, uint32_t k, uint64_t rows,
                     const float* wt, const float* bias, const float* pre_bias, uint32_t m,
                     uint32_t pre, uint32_t act, float* out, uint32_t out_pitch, float* out2,
                     float out2_scale, cudaStream_t st, const float* row_scale) {
  if (rows == 0) return;
  TcArgs a{};
  a.row_scale = row_scale;
  a.rows = rows;
  a.k = k;
  a.n_kb = (k + BK - 1) / BK;
  a.m = m;
  a.out_pitch = out_pitch;
  a.pre = pre;
  a.act = act;
  a.bias = bias;
  a.pre_bias = pre_bias;
  a.out = out;
  a.out2 = out2;
  a.out2_scale = out2_scale;
  const uint32_t kpad = a.n_kb * BK;
  const uint32_t np = (m + 15) / 16 * 16;
  // four epilogue groups for short-K GEMMs (the heads: the epilogue binds),
  // two (NP <= 48) or one otherwise
  static const uint32_t g4_kb = [] {
    const char* e = std::getenv("MGG_TC_G4_KB");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 2u;
  }();
  const bool g4 = a.n_kb <= g4_kb;
  switch (np) {
    case 16: g4 ? run_tc<16, false, 4>(in, in_pitch, wt, kpad, nullptr, a, st)
                : run_tc<16, false, 2>(in, in_pitch, wt, kpad, nullptr, a, st); break;
    case 32: g4 ? run_tc<32, false, 4>(in, in_pitch, wt, kpad, nullptr, a, st)
                : run_tc<32, false, 2>(in, in_pitch, wt, kpad, nullptr, a, st); break;
    case 48: {
      static const int eg48 = [] {
        const char* e = std::getenv("MGG_TC_EG48");
        // measured: 4 groups (80 registers, 16 B of spill) beat 3 once the
        // staging selects were gone (products head 0.164 -> 0.147 ms)
        return e ? std::atoi(e) : 4;
      }();
      if (!g4) run_tc<48, false, 2>(in, in_pitch, wt, kpad, nullptr, a, st);
      else if (eg48 == 4) run_tc<48, false, 4>(in, in_pitch, wt, kpad, nullptr, a, st);
      else run_tc<48, false, 3>(in, in_pitch, wt, kpad, nullptr, a, st);
      break;
    }
    case 64: run_tc<64, false, 1>(in, in_pitch, wt, kpad, nullptr, a, st); break;
    default: throw Status{MGG_E_CONFIG, "gemm_tc: unsupported width"};
  }
}

bool gemm_tc_chain_supported(uint32_t k, uint32_t m1, uint32_t m) {
  // O = m1 columns must be exactly the second GEMM's padded K (whole 32-wide
  // k-blocks in TMEM), and both products share NP
  const uint32_t np = (m + 15) / 16 * 16;
  return gemm_tc_supported(k, m) && m1 == np && np % BK == 0 && m1 <= 64;
}

void launch_dense_tc_chain(const float* in, uint32_t in_pitch, uint32_t k, uint64_t rows,
                           const float* wt1, const float* bias1, uint32_t m1,
                           const float* pre_bias, uint32_t pre, const float* wt2,
                           uint32_t m, float* out, uint32_t out_pitch, float* out2,
                           float out2_scale, cudaStream_t st) {
  if (rows == 0) return;
  TcArgs a{};
  a.rows = rows;
  a.k = k;
  a.n_kb = (k + BK - 1) / BK;
  a.m = m;
  a.m1 = m1;
  a.out_pitch = out_pitch;
  a.pre = pre;
  a.act = 0;
  a.bias = nullptr;
  a.bias1 = bias1;
  a.pre_bias = pre_bias;
  a.out = out;
  a.out2 = out2;
  a.out2_scale = out2_scale;
  const uint32_t kpad = a.n_kb * BK;
  switch ((m + 15) / 16 * 16) {
    case 32: run_tc<32, true, 2>(in, in_pitch, wt1, kpad, wt2, a, st); break;
    case 64: run_tc<64, true, 1>(in, in_pitch, wt1, kpad, wt2, a, st); break;
    default: throw Status{MGG_E_CONFIG, "gemm_tc chain: unsupported width"};
  }
}

}  // namespace mgg::dev
