// fp64_peak.cu — measurement helper for bench.py (not part of the LOFP method): the
// B200's FP64 issue ceiling, measured, so that the roofline denominator of the path
// enumeration kernel is a number taken on the same box rather than a datasheet value.
//
// Each thread runs 16 independent DFMA chains (enough ILP to cover the pipe latency);
// every grid covers all SMs at full occupancy.  The result is DFMA lane-instructions per
// second (one DFMA = 2 flops).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
__global__ void __launch_bounds__(256) dfma_chains(double *out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = (double)(threadIdx.x + i) * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}
}  // namespace

extern "C" {
// Returns DFMA lane-instructions per second measured over `reps` launches (best), or a
// negative value on a CUDA error.  `sm_count` receives the number of SMs.
double lofp_probe_fp64_dfma_rate(int reps, int *sm_count) {
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1.0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dfma_chains, 256, 0) != cudaSuccess) return -1.0;
  if (sm_count) *sm_count = sms;
  double *buf = nullptr;
  if (cudaMalloc(&buf, 16) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, grid = sms * per_sm;
  dfma_chains<<<grid, 256>>>(buf, 64, 1.0000001, 1e-12);  // warm-up
  double best = 0.0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    dfma_chains<<<grid, 256>>>(buf, iters, 1.0000001, 1e-12);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    double rate = (double)grid * 256.0 * iters * 16.0 / (ms * 1e-3);
    if (rate > best) best = rate;
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return e == cudaSuccess ? best : -1.0;
}
}
