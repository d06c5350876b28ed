// Does splitting a random-row gather between the two dies raise the L2 hit
// rate? (tools/l2_capacity_sweep.py: uniform random 64-B gathers from every
// SM see an effective L2 of only ~40-46 MB of the 126 MB.)
//
// 1. SM -> die map: block 0 warms 64 lines 2 KB apart, every block times the
//    same lines (32 dependent ld.cg each); the latency vector correlates
//    positively with block 0's on block 0's die and negatively on the other
//    (tools/l2_die_probe.cu showed the split: 72 / 76 SMs).
// 2. Row -> home die: for every 2 KB chunk of the table one warp on block
//    0's die times one line of it; near (below the median) = block 0's die.
// 3. Gathers, TABLE_MB table of 64-B rows, 60M gathers per launch, modes:
//      0 uniform  : every SM draws rows from the whole table
//      1 idx-half : die-0 SMs draw rows [0, N/2), die-1 SMs [N/2, N)
//      2 home     : each SM draws rows whose 2 KB chunk is homed on its die
//    Printed: ms per launch (CUDA events, median of 5) per mode; run under
//    ncu for the L2 hit rate.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_split_probe tools/l2_split_probe.cu
// usage: l2_split_probe TABLE_MB [mode]   (mode given: only that mode, 2 launches, for ncu)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int kLines = 64, kRep = 32;
constexpr size_t kChunk = 2048;

__device__ unsigned g_arrive;

__device__ __forceinline__ unsigned chase(const char* p, unsigned& v) {
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

// one warp per block, grid = #SMs (co-resident): smid + latency of 64 lines
__global__ void die_map(const char* lines, unsigned* lat, int* smid_of_block) {
  if (threadIdx.x) return;
  int smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  smid_of_block[blockIdx.x] = smid;
  unsigned v = 0x01010101u;
  if (blockIdx.x == 0)
    for (int i = 0; i < kLines; ++i) chase(lines + i * kChunk, v);
  atomicAdd(&g_arrive, 1u);
  while (atomicAdd(&g_arrive, 0u) < gridDim.x) {
  }
  for (int i = 0; i < kLines; ++i) lat[blockIdx.x * kLines + i] = chase(lines + i * kChunk, v);
  if (v != 0x01010101u) lat[0] = v;
}

// chunk latencies from SMs of die 0 only (blocks whose SM is on die 0 work)
__device__ unsigned long long g_next_chunk;
__global__ void chunk_home(const char* table, size_t nchunks, const int* die_of_sm,
                           unsigned* lat) {
  int smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (die_of_sm[smid] != 0) return;
  if (threadIdx.x & 31) return;
  unsigned v = 0x01010101u;
  for (;;) {  // chunks dealt dynamically to the die-0 warps
    const unsigned long long c = atomicAdd(&g_next_chunk, 1ull);
    if (c >= nchunks) break;
    lat[c] = chase(table + c * kChunk, v);
  }
  if (v != 0x01010101u) lat[0] = v;
}

__device__ __forceinline__ unsigned mix(unsigned x) {  // cheap 32-bit hash
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  return x ^ (x >> 16);
}

// 4 lanes per 64-B row, 8 rows per warp step, 4 steps in flight
__global__ void __launch_bounds__(256) gather(const float4* table, size_t rows, size_t n,
                                              int mode, const int* die_of_sm,
                                              const unsigned* home_chunks, const size_t* home_n,
                                              float* sink) {
  int smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const int die = die_of_sm[smid];
  const int lane = threadIdx.x & 31, sub = lane >> 2, v = lane & 3;
  const size_t warp = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
  const size_t nw = (gridDim.x * size_t(blockDim.x)) >> 5;
  const size_t half = rows / 2;
  const size_t rows_per_chunk = kChunk / 64;
  float4 acc = make_float4(0, 0, 0, 0);
  for (size_t base = warp * 32; base < n; base += nw * 32) {
    float4 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned h = mix(static_cast<unsigned>(base + u * 8 + sub));
      size_t r;
      if (mode == 0) {
        r = __umulhi(h, static_cast<unsigned>(rows));
      } else if (mode == 1) {
        r = __umulhi(h, static_cast<unsigned>(half)) + (die ? half : 0);
      } else {
        const size_t c = home_chunks[die * rows + __umulhi(h, static_cast<unsigned>(home_n[die]))];
        r = c * rows_per_chunk + (h & (rows_per_chunk - 1));
      }
      t[u] = __ldcg(table + r * 4 + v);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc.x += t[u].x, acc.y += t[u].y, acc.z += t[u].z, acc.w += t[u].w;
  }
  if (acc.x == 1234.5f) sink[0] = acc.y + acc.z + acc.w;
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? std::atoi(argv[1]) : 160;
  const int only = argc > 2 ? std::atoi(argv[2]) : -1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t bytes = mb << 20, rows = bytes / 64, nchunks = bytes / kChunk;
  char *table, *lines;
  unsigned *lat, *clat, *home_chunks;
  int *smid_of_block, *die_of_sm;
  size_t* home_n;
  float* sink;
  cudaMalloc(&table, bytes);
  cudaMemset(table, 1, bytes);
  cudaMalloc(&lines, kLines * kChunk);
  cudaMemset(lines, 1, kLines * kChunk);
  cudaMalloc(&lat, sms * kLines * 4);
  cudaMalloc(&smid_of_block, sms * 4);
  cudaMalloc(&die_of_sm, 1024 * 4);
  cudaMalloc(&clat, nchunks * 4);
  cudaMalloc(&home_chunks, 2 * rows * 4);
  cudaMalloc(&home_n, 2 * sizeof(size_t));
  cudaMalloc(&sink, 4);
  unsigned zero = 0;
  cudaMemcpyToSymbol(g_arrive, &zero, 4);
  die_map<<<sms, 32>>>(lines, lat, smid_of_block);
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;
  std::vector<unsigned> L(sms * kLines);
  std::vector<int> S(sms), D(1024, 0);
  cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(S.data(), smid_of_block, sms * 4, cudaMemcpyDeviceToHost);
  int n0 = 0;
  for (int b = 0; b < sms; ++b) {
    double ma = 0, mb2 = 0, sab = 0;
    for (int i = 0; i < kLines; ++i) ma += L[i], mb2 += L[b * kLines + i];
    ma /= kLines, mb2 /= kLines;
    for (int i = 0; i < kLines; ++i) sab += (L[i] - ma) * (L[b * kLines + i] - mb2);
    D[S[b]] = sab >= 0 ? 0 : 1;
    n0 += sab >= 0;
  }
  cudaMemcpy(die_of_sm, D.data(), 1024 * 4, cudaMemcpyHostToDevice);
  unsigned long long z64 = 0;
  cudaMemcpyToSymbol(g_next_chunk, &z64, 8);
  chunk_home<<<sms * 4, 256>>>(table, nchunks, die_of_sm, clat);
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  std::vector<unsigned> CL(nchunks);
  cudaMemcpy(CL.data(), clat, nchunks * 4, cudaMemcpyDeviceToHost);
  std::vector<unsigned> sorted = CL;
  std::nth_element(sorted.begin(), sorted.begin() + nchunks / 2, sorted.end());
  const unsigned med = sorted[nchunks / 2];
  std::vector<unsigned> hc(2 * rows, 0);
  size_t hn[2] = {0, 0};
  for (size_t c = 0; c < nchunks; ++c) {
    const int d = CL[c] < med ? 0 : 1;
    hc[d * rows + hn[d]++] = static_cast<unsigned>(c);
  }
  cudaMemcpy(home_chunks, hc.data(), hc.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(home_n, hn, sizeof(hn), cudaMemcpyHostToDevice);
  const size_t n = 60000000;
  std::printf("{\"table_MB\": %zu, \"die0_sms\": %d, \"die1_sms\": %d, \"chunks_die0\": %zu, "
              "\"chunks_die1\": %zu, \"chunk_lat_median\": %u",
              mb, n0, sms - n0, hn[0], hn[1], med);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    if (only >= 0 && mode != only) continue;
    std::vector<float> ms;
    const int reps = only >= 0 ? 2 : 6;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(e0);
      gather<<<sms * 8, 256>>>(reinterpret_cast<const float4*>(table), rows, n, mode, die_of_sm,
                               home_chunks, home_n, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float t = 0;
      cudaEventElapsedTime(&t, e0, e1);
      if (r) ms.push_back(t);
    }
    std::sort(ms.begin(), ms.end());
    const float m = ms[ms.size() / 2];
    std::printf(", \"mode%d_ms\": %.4f, \"mode%d_rows_TBps\": %.2f", mode, m, mode,
                n * 64.0 / (m * 1e-3) / 1e12);
  }
  std::printf("}\n");
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
