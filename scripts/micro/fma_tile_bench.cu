// Microbenchmark: the unit kernel's warp tile (8 complex X per lane in registers x a 256-value
// Y slice in shared memory, four Y values loaded ahead of their 128 DFMA) at the unit
// kernel's occupancy (2 blocks x 256 threads per SM), no list building or loads.  Reports
// DFMA lane-instructions per second.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kKX = 8, kYT = 256;

#define CFMA(v)                                     \
  _Pragma("unroll") for (int r = 0; r < kKX; ++r) { \
    acc[r].x = fma(x[r].x, (v).x, acc[r].x);        \
    acc[r].y = fma(x[r].x, (v).y, acc[r].y);        \
    acc[r].x = fma(-x[r].y, (v).y, acc[r].x);       \
    acc[r].y = fma(x[r].y, (v).x, acc[r].y);        \
  }

__global__ void __launch_bounds__(256, 2) tile_kernel(int reps, double2 *out) {
  __shared__ double2 sY[8 * kYT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *sW = sY + warp * kYT;
  for (int i = lane; i < kYT; i += 32) sW[i] = make_double2(1e-3 * i, -2e-3 * i);
  double2 x[kKX], acc[kKX];
  for (int r = 0; r < kKX; ++r) {
    x[r] = make_double2(0.5 + lane * 1e-3 + r, 0.25 - r * 1e-3);
    acc[r] = make_double2(0.0, 0.0);
  }
  __syncwarp();
  for (int it = 0; it < reps; ++it) {
    for (int y = 0; y + 3 < kYT; y += 4) {
      const double2 v0 = sW[y], v1 = sW[y + 1], v2 = sW[y + 2], v3 = sW[y + 3];
      CFMA(v0) CFMA(v1) CFMA(v2) CFMA(v3)
    }
  }
  double2 s = make_double2(0, 0);
  for (int r = 0; r < kKX; ++r) { s.x += acc[r].x; s.y += acc[r].y; }
  if (s.x == 1.2345) out[0] = s;  // keep the work
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double2 *out;
  cudaMalloc(&out, 16);
  const int reps = 2000, grid = 2 * nsm;
  tile_kernel<<<grid, 256>>>(10, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tile_kernel<<<grid, 256>>>(reps, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = (double)grid * 256 * reps * kYT * kKX * 4;
  printf("{\"tile_dfma_per_s\": %.4e, \"paths_per_s_equiv\": %.4e, \"ms\": %.3f}\n", dfma / (ms * 1e-3),
         dfma / 4 / (ms * 1e-3), ms);
  return 0;
}
