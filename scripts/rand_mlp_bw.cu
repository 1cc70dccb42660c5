// Per-SM memory-level-parallelism probe: random 256-byte line reads over a 16 GB buffer,
// W warps per SM each with L independent line loads in flight (LDG path), and the same
// with each warp's lines fetched by cp.async.bulk (TMA path) into shared memory.
// Answers: is random-line bandwidth capped by lines in flight per SM, and does the bulk
// path raise the cap?  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

template <int L>
__global__ void k_ldg(const double *buf, uint64_t nlines, uint64_t iters, double *sink) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (uint64_t it = 0; it < iters; ++it) {
    double v[L];
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const uint64_t c = mix((it * nw + warp) * L + k) & (nlines - 1);
      v[k] = __ldcg(buf + (c << 5) + lane);
    }
#pragma unroll
    for (int k = 0; k < L; ++k) acc += v[k];
  }
  if (acc == 1.2345) sink[0] = acc;
}

template <int L>
__global__ void k_bulk(const double *buf, uint64_t nlines, uint64_t iters, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double *stage = reinterpret_cast<double *>(sm + (size_t)wid * (L * 256 + 16));
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)wid * (L * 256 + 16) + L * 256);
  const unsigned ba = (unsigned)__cvta_generic_to_shared(bar);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  double acc = 0.0;
  unsigned phase = 0;
  for (uint64_t it = 0; it < iters; ++it) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(L * 256) : "memory");
#pragma unroll
      for (int k = 0; k < L; ++k) {
        const uint64_t c = mix((it * nw + warp) * L + k) & (nlines - 1);
        const unsigned d = (unsigned)__cvta_generic_to_shared(stage + k * 32);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                     ::"r"(d), "l"(buf + (c << 5)), "r"(ba) : "memory");
      }
    }
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(ba), "r"(phase) : "memory");
    phase ^= 1u;
#pragma unroll
    for (int k = 0; k < L; ++k) acc += stage[k * 32 + lane];
    __syncwarp();
  }
  if (acc == 1.2345) sink[0] = acc;
}

template <int L>
static void run(const double *buf, double *sink, uint64_t nlines, int warps_per_sm, bool bulk) {
  const int threads = warps_per_sm >= 8 ? 256 : warps_per_sm * 32;
  const int blocks = 148 * (warps_per_sm * 32 / threads);
  const uint64_t nw = (uint64_t)blocks * threads / 32;
  const uint64_t iters = (4ull << 30) / (nw * L * 256);
  const size_t smem = (size_t)(threads / 32) * (L * 256 + 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    if (bulk) {
      cudaFuncSetAttribute(k_bulk<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_bulk<L><<<blocks, threads, smem>>>(buf, nlines, iters, sink);
    } else
      k_ldg<L><<<blocks, threads>>>(buf, nlines, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double gb = (double)iters * nw * L * 256 / 1e9;
  printf("{\"path\": \"%s\", \"warps_per_sm\": %d, \"lines_per_warp\": %d, \"lines_in_flight_per_sm\": %d, \"GBps\": %.0f, \"err\": %d}\n",
         bulk ? "bulk" : "ldg", warps_per_sm, L, warps_per_sm * L, gb / best * 1e3, (int)cudaGetLastError());
  fflush(stdout);
}

int main() {
  const uint64_t bytes = 16ull << 30;
  double *buf, *sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 0, bytes);
  const uint64_t nlines = bytes / 256;
  for (int bulk = 0; bulk < 2; ++bulk)
    for (int w : {4, 8, 16, 32, 64}) {
      run<2>(buf, sink, nlines, w, bulk);
      run<4>(buf, sink, nlines, w, bulk);
      run<8>(buf, sink, nlines, w, bulk);
      run<16>(buf, sink, nlines, w, bulk);
      if (w <= 32) run<32>(buf, sink, nlines, w, bulk);
    }
  return 0;
}
