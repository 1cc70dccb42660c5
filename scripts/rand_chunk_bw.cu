// Random-chunk DRAM bandwidth probe: warps read (or write) CHUNK-byte contiguous pieces
// at pseudo-random CHUNK-aligned offsets of a buffer much larger than L2, 8 independent
// 256-byte line loads in flight per warp.  Answers: what does DRAM deliver for the
// batched kernels' access pattern (random 256-byte lines) vs 512 B / 1 KB / ... pieces?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o rand_chunk_bw rand_chunk_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

template <int MODE>   // 0 read, 1 write, 2 read + write (different random chunks)
__global__ void k_probe(double *buf, uint64_t nchunks, int lines_per_chunk, uint64_t iters, double *sink) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  const int lsh = 31 - __clz(lines_per_chunk);
  // each iteration: 8 lines = 8 / lines_per_chunk chunks (or one chunk of >= 8 lines in pieces)
  for (uint64_t it = 0; it < iters; ++it) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint64_t lineno = (it * nw + warp) * 8 + k;
      const uint64_t c = mix(lineno >> lsh) & (nchunks - 1);
      const uint64_t off = (((c << lsh) + (lineno & (lines_per_chunk - 1))) << 5) + lane;
      if (MODE == 0 || MODE == 2) v[k] = __ldcg(buf + off);
      if (MODE == 1) __stcg(buf + off, (double)it);
      if (MODE == 2) {
        const uint64_t c2 = mix((lineno >> lsh) + 0x9e3779b97f4a7c15ULL) & (nchunks - 1);
        __stcg(buf + ((((c2 << lsh) + (lineno & (lines_per_chunk - 1))) << 5) + lane), (double)it);
      }
    }
    if (MODE != 1)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k];
  }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  const uint64_t bytes = 16ull << 30;
  double *buf, *sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 0, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 8, threads = 256;   // 64 warps/SM, 8 lines in flight each
  const uint64_t nw = (uint64_t)blocks * threads / 32;
  for (int mode = 0; mode < 3; ++mode)
    for (int chunk = 256; chunk <= 8192; chunk *= 2) {
      const int lpc = chunk / 256;
      const uint64_t nchunks = bytes / chunk;
      const uint64_t iters = (8ull << 30) / (nw * 8 * 256);   // 8 GB touched per launch
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) k_probe<0><<<blocks, threads>>>(buf, nchunks, lpc, iters, sink);
        if (mode == 1) k_probe<1><<<blocks, threads>>>(buf, nchunks, lpc, iters, sink);
        if (mode == 2) k_probe<2><<<blocks, threads>>>(buf, nchunks, lpc, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const double gb = (double)iters * nw * 8 * 256 * (mode == 2 ? 2 : 1) / 1e9;
      printf("{\"mode\": \"%s\", \"chunk\": %d, \"ms\": %.3f, \"GBps\": %.1f}\n",
             mode == 0 ? "read" : mode == 1 ? "write" : "read+write", chunk, best, gb / best * 1e3);
      fflush(stdout);
    }
  return cudaGetLastError() != cudaSuccess;
}
