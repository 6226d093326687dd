// Measured peaks the bench's rooflines need beside MEASURED_PEAKS.json
// ("the builder must measure" the FP32 FFMA peak; the L2 read
// bandwidth for W_hh that stays L2-resident).  Built by tools/peak_probe.py.
#include <cuda_runtime.h>
#include <stdint.h>

// 8 independent FMA chains per thread, long enough to amortise launch cost
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678f) out[blockIdx.x] = s;  // never true: keeps the chains live
}

// every thread streams 16-B vectors of `buf` (bytes), `reps` times
__global__ void read_kernel(const uint4* __restrict__ buf, size_t n16, int reps, uint32_t* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
      uint4 v;
      asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + i));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

extern "C" {
// FP32 FFMA throughput in TFLOP/s (2 flops per FMA), best of `trials`
float probe_ffma_tflops(int trials) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 0.f;
  ffma_kernel<<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f);
  for (int t = 0; t < trials; ++t) {
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    const float tf = (float)(flops / (ms * 1e-3) / 1e12);
    if (tf > best) best = tf;
  }
  cudaFree(out);
  return best;
}

// read bandwidth (GB/s) over a buffer of `bytes`, re-read `reps` times per launch:
// 64 MiB stays in the 126 MB L2 (the c4 W_hh working set), 4 GiB does not
float probe_read_gbs(size_t bytes, int reps, int trials) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* buf;
  uint32_t* sink;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return -1.f;
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t n16 = bytes / 16;
  read_kernel<<<sms * 4, 512>>>(buf, n16, 1, sink);
  float best = 0.f;
  for (int t = 0; t < trials; ++t) {
    cudaEventRecord(e0);
    read_kernel<<<sms * 4, 512>>>(buf, n16, reps, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const float gbs = (float)((double)bytes * reps / (ms * 1e-3) / 1e9);
    if (gbs > best) best = gbs;
  }
  cudaFree(buf);
  cudaFree(sink);
  return best;
}
}
