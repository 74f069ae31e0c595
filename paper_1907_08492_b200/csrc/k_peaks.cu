// Machine-characterisation kernels (the paper's MKL dgemm / STREAM roles,
// PAPER.md:814-849): the fp64 DFMA roof and a streaming
// copy/read bandwidth, measured with CUDA events on the caller's stream.
#include <cuda_runtime.h>

#include <cstdint>

namespace dgb {
namespace {

constexpr int kChains = 8;

__global__ void k_dfma(double* sink, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1.2345) sink[threadIdx.x] = s;   // never true; keeps the chains alive
}

// FP64 tensor-core throughput (DMMA, mma.sync m8n8k4 f64: 256 FMA per warp instruction),
// KC independent accumulator chains per warp; MIX > 0 also runs MIX DFMA chains per thread
// in the same loop, to see whether the two share a pipe
template <int KC, int MIX>
__global__ void k_dmma(double* sink, int iters, double a, double b) {
  double acc[KC][2];
#pragma unroll
  for (int c = 0; c < KC; ++c) acc[c][0] = acc[c][1] = threadIdx.x * 1e-9 + c;
  double x[MIX > 0 ? MIX : 1];
#pragma unroll
  for (int c = 0; c < (MIX > 0 ? MIX : 1); ++c) x[c] = threadIdx.x * 1e-9 + c;
  const double av = a + threadIdx.x * 1e-12, bv = b - threadIdx.x * 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int c = 0; c < KC; ++c)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1])
                     : "d"(av), "d"(bv));
      if constexpr (MIX > 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int c = 0; c < MIX; ++c) x[c] = fma(x[c], a, b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < KC; ++c) s += acc[c][0] + acc[c][1];
#pragma unroll
  for (int c = 0; c < (MIX > 0 ? MIX : 1); ++c) s += x[c];
  if (s == 1.2345) sink[threadIdx.x] = s;
}

__global__ void k_copy(const double2* __restrict__ in, double2* __restrict__ out, int64_t n2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void k_read(const double2* __restrict__ in, double* sink, int64_t n2) {
  double acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = in[i];
    acc += v.x + v.y;
  }
  if (acc == 1.2345) sink[0] = acc;
}

}  // namespace

// kind 0: fp64 FMA TFLOP/s; 1: copy GB/s (read + write bytes); 2: read-only GB/s;
// 3: fp64 tensor-core (DMMA) TFLOP/s; 4: DMMA and DFMA chains interleaved, total TFLOP/s
cudaError_t measure_plane_probe(int n, double* value, cudaStream_t s);   // k_probe_plane.cu

cudaError_t measure_peak(int kind, double* value, cudaStream_t s) {
  if (kind >= 13 && kind <= 18) return measure_plane_probe(kind - 10, value, s);
  if (kind >= 23 && kind <= 26) return measure_plane_probe(kind - 10, value, s);   // with neighbour traffic
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaError_t err = cudaSuccess;
  float best_ms = 1e30f;
  double work = 0;
  if (kind == 3 || kind == 4) {
    double* sink;
    err = cudaMalloc(&sink, 1024 * sizeof(double));
    if (err != cudaSuccess) return err;
    const int blocks = 148 * 8, threads = 256, iters = 2048;
    constexpr int KC = 4, MIX = 8;
    // DMMA: 512 FLOP per warp instruction; DFMA: 2 FLOP per thread instruction
    work = (double)blocks * (threads / 32) * iters * 4 * KC * 512.0;
    if (kind == 4) work += 2.0 * blocks * threads * (double)iters * 4 * 4 * MIX;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0, s);
      if (kind == 3)
        k_dmma<KC, 0><<<blocks, threads, 0, s>>>(sink, iters, 0.999999, 1e-7);
      else
        k_dmma<KC, MIX><<<blocks, threads, 0, s>>>(sink, iters, 0.999999, 1e-7);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best_ms) best_ms = ms;
    }
    err = cudaGetLastError();
    cudaFree(sink);
    *value = work / (best_ms * 1e-3) / 1e12;
  } else if (kind == 0) {
    double* sink;
    err = cudaMalloc(&sink, 1024 * sizeof(double));
    if (err != cudaSuccess) return err;
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    work = 2.0 * blocks * threads * (double)iters * 16 * kChains;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0, s);
      k_dfma<<<blocks, threads, 0, s>>>(sink, iters, 0.999999, 1e-7);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best_ms) best_ms = ms;
    }
    err = cudaGetLastError();
    cudaFree(sink);
    *value = work / (best_ms * 1e-3) / 1e12;
  } else {
    const int64_t bytes = 2LL << 30;   // 2 GiB per buffer (>> 126 MB L2)
    double2 *a, *b;
    err = cudaMalloc(&a, bytes);
    if (err != cudaSuccess) return err;
    err = cudaMalloc(&b, bytes);
    if (err != cudaSuccess) {
      cudaFree(a);
      return err;
    }
    cudaMemsetAsync(a, 0, bytes, s);
    cudaMemsetAsync(b, 0, bytes, s);
    const int64_t n2 = bytes / 16;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0, s);
      if (kind == 1)
        k_copy<<<148 * 16, 512, 0, s>>>(a, b, n2);
      else
        k_read<<<148 * 16, 512, 0, s>>>(a, (double*)b, n2);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best_ms) best_ms = ms;
    }
    err = cudaGetLastError();
    work = (kind == 1 ? 2.0 : 1.0) * bytes;
    cudaFree(a);
    cudaFree(b);
    *value = work / (best_ms * 1e-3) / 1e9;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return err;
}

}  // namespace dgb
