// probe.cu -- measured FP64 lane peak of the device (the roofline denominator
// of the sweep).  MEASURED_PEAKS.json carries HBM and
// bf16 figures only; the sweep is bound by the FP64 pipe, so the
// bench measures that pipe's throughput on the same GPU, in the same process,
// with the same counting rule as the sweep's roofline: one DADD / DMUL / DFMA
// thread-instruction = one lane-op.
//
// Kernel: every thread runs kChains independent DFMA chains (x = x * a + b,
// a = 1 - 2^-30, so values stay bounded and never denormal), unrolled, at full
// occupancy (1024-thread blocks, 2 per SM = 64 warps/SM): enough independent
// work per SMSP to hide the DFMA latency, so the time is set by the FP64 issue
// rate alone.  Result: lane-ops/s = threads x iters x kChains / seconds.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(1024, 2) fp64_peak_kernel(int iters, double a, double b, double* sink) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = 1.0 + (threadIdx.x + c) * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) *sink = s;  // never true; keeps the chains live
}

}  // namespace

// Measured FP64 lane-op throughput (ops/s) on `device`: best of `reps` timed
// launches after one warm-up.  Returns cudaSuccess or the first CUDA error.
extern "C" cudaError_t libperm_probe_fp64_peak(int device, int reps, double* ops_per_s, double* ms_best) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return e;
  int sms = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device)) != cudaSuccess) return e;
  double* sink = nullptr;
  if ((e = cudaMalloc(&sink, sizeof(double))) != cudaSuccess) return e;
  cudaStream_t st;
  cudaEvent_t e0, e1;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 2 * sms, threads = 1024, iters = 4096;
  const double a = 1.0 - 1.0 / (1 << 30), b = 1.0 / (1 << 20);
  fp64_peak_kernel<<<grid, threads, 0, st>>>(iters, a, b, sink);  // warm-up / clock ramp
  float best = 1e30f;
  for (int r = 0; r < (reps > 0 ? reps : 5); ++r) {
    cudaEventRecord(e0, st);
    fp64_peak_kernel<<<grid, threads, 0, st>>>(iters, a, b, sink);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaFree(sink);
  if (e != cudaSuccess) return e;
  const double ops = (double)grid * threads * iters * 16.0 * kChains;
  *ops_per_s = ops / (best * 1e-3);
  if (ms_best) *ms_best = best;
  return cudaSuccess;
}
