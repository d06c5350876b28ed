// L2 die topology probe (B200 is two dies; the L2 is split between them).
//
// Question: does a die's L2 keep its own copy of lines homed on the other
// die (so a table read by every SM occupies both halves and the effective
// capacity for it is ~63 MB, not 126 MB)? And which SMs sit on which die?
//
// One warp per CTA, 148 CTAs (one per SM, all co-resident). Block 0 warms
// every probe line (ld.global.cg), grid barrier, then block b times its own
// 64 lines (2 KB apart, so their home die varies ~Bernoulli(0.5)), one
// dependent ld.global.cg at a time. Then the same again with block 0's lines
// read a second time by block b after block b has already touched them.
//   * No duplication: block 0 itself sees a bimodal pattern (near ~234 /
//     far ~262 cycles), every SM's pattern equals block 0's or its inverse.
//   * Duplication: block 0 sees all near (its die now holds copies); SMs on
//     block 0's die see all near, SMs on the other die see far for the lines
//     homed on block 0's die.
// Output: one JSON object (per-block smid, near/far counts, mean latency and
// the latency vector's correlation with block 0's).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/l2_die_probe tools/l2_die_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int kLines = 64;
constexpr size_t kStride = 2048;  // bytes between probe lines

__device__ unsigned g_arrive;

__device__ void grid_sync(unsigned n, unsigned phase) {
  __syncwarp();
  if (threadIdx.x == 0) {
    atomicAdd(&g_arrive, 1u);
    while (atomicAdd(&g_arrive, 0u) < n * phase) {
    }
  }
  __syncwarp();
}

// 32 dependent ld.global.cg of the same line (the address carries the loaded
// value, which is the memset pattern 0x01010101, minus itself): cycles / 32.
// A clock read that the scheduler hoists costs at most one load of error.
constexpr int kRep = 32;
// `v` carries over from the previous call, so consecutive lines' chains are
// serialised too.
__device__ __forceinline__ unsigned lat_of(const char* p, unsigned& v) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
#pragma unroll
  for (int k = 0; k < kRep; ++k)
    asm volatile(
        "{\n\t.reg .u32 o;\n\t.reg .u64 a;\n\tsub.u32 o, %1, 16843009;\n\t"
        "cvt.u64.u32 a, o;\n\tadd.u64 a, a, %2;\n\tld.global.cg.u32 %0, [a];\n\t}"
        : "=r"(v)
        : "r"(v), "l"(p)
        : "memory");
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
  return static_cast<unsigned>((t1 - t0) / kRep);
}

__global__ void probe(const char* buf, unsigned* lat, unsigned* lat0again, int* smid_out,
                      unsigned* sink) {
  int smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const unsigned n = gridDim.x;
  unsigned acc = 0x01010101u;  // the chained load value (memset pattern)
  if (threadIdx.x == 0) {
    smid_out[blockIdx.x] = smid;
    if (blockIdx.x == 0)  // warm every block's lines from block 0's SM
      for (unsigned i = 0; i < n * kLines; ++i) lat_of(buf + size_t(i) * kStride, acc);
  }
  grid_sync(n, 1);
  if (threadIdx.x == 0) {
    const char* mine = buf + size_t(blockIdx.x) * kLines * kStride;
    for (int i = 0; i < kLines; ++i) lat[blockIdx.x * kLines + i] = lat_of(mine + i * kStride, acc);
  }
  grid_sync(n, 2);
  // block 0's own lines (warmed and re-read by block 0 only), now read by
  // every block in turn — a second look at the same addresses from all SMs
  for (unsigned b = 0; b < n; ++b) {
    if (blockIdx.x == b && threadIdx.x == 0)
      for (int i = 0; i < kLines; ++i) lat0again[b * kLines + i] = lat_of(buf + i * kStride, acc);
    grid_sync(n, 3 + b);
  }
  if (acc != 0x01010101u) sink[0] = acc;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t bytes = size_t(sms) * kLines * kStride;
  char* buf;
  unsigned *lat, *lat0, *sink;
  int* smid;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaMalloc(&lat, sms * kLines * 4);
  cudaMalloc(&lat0, sms * kLines * 4);
  cudaMalloc(&smid, sms * 4);
  cudaMalloc(&sink, 4);
  unsigned zero = 0;
  cudaMemcpyToSymbol(g_arrive, &zero, 4);
  probe<<<sms, 32>>>(buf, lat, lat0, smid, sink);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<unsigned> L(sms * kLines), L0(sms * kLines);
  std::vector<int> S(sms);
  cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(L0.data(), lat0, L0.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(S.data(), smid, sms * 4, cudaMemcpyDeviceToHost);
  auto corr = [&](const unsigned* a, const unsigned* b) {
    double ma = 0, mb = 0;
    for (int i = 0; i < kLines; ++i) ma += a[i], mb += b[i];
    ma /= kLines, mb /= kLines;
    double sab = 0, saa = 0, sbb = 0;
    for (int i = 0; i < kLines; ++i) {
      sab += (a[i] - ma) * (b[i] - mb);
      saa += (a[i] - ma) * (a[i] - ma);
      sbb += (b[i] - mb) * (b[i] - mb);
    }
    return saa > 0 && sbb > 0 ? sab / std::sqrt(saa * sbb) : 0.0;
  };
  std::printf("{\"sms\": %d, \"lines_per_sm\": %d, \"stride\": %zu, \"blocks\": [", sms, kLines, kStride);
  for (int b = 0; b < sms; ++b) {
    const unsigned* v = &L[b * kLines];
    const unsigned* w = &L0[b * kLines];
    double m = 0, m0 = 0;
    unsigned lo = ~0u, hi = 0;
    for (int i = 0; i < kLines; ++i) m += v[i], m0 += w[i], lo = std::min(lo, v[i]), hi = std::max(hi, v[i]);
    std::printf("%s{\"block\": %d, \"smid\": %d, \"own_mean\": %.1f, \"own_min\": %u, \"own_max\": %u, "
                "\"own_corr_block0\": %.3f, \"block0_lines_mean\": %.1f, \"block0_lines_corr_block0\": %.3f, "
                "\"own\": [",
                b ? ", " : "", b, S[b], m / kLines, lo, hi, corr(v, &L[0]), m0 / kLines,
                corr(w, &L0[0]));
    for (int i = 0; i < kLines; ++i) std::printf("%s%u", i ? "," : "", v[i]);
    std::printf("], \"b0lines\": [");
    for (int i = 0; i < kLines; ++i) std::printf("%s%u", i ? "," : "", w[i]);
    std::printf("]}");
  }
  std::printf("]}\n");
  return 0;
}
