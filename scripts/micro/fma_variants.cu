// Variants of the warp tile loop (see fma_tile_bench.cu): X values per lane KX, blocks per SM
// MINB, Y loads ahead UNR, FMA order ORD (0: per r four FMAs; 1: all first halves, then all
// second halves).  Prints DFMA lane-instructions per second for each.
#include <cstdio>
#include <cuda_runtime.h>

template <int KX, int UNR, int ORD>
__device__ __forceinline__ void cfma(double2 (&acc)[KX], const double2 (&x)[KX], const double2 *v) {
  if (ORD == 0) {
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int r = 0; r < KX; ++r) {
        acc[r].x = fma(x[r].x, v[u].x, acc[r].x);
        acc[r].y = fma(x[r].x, v[u].y, acc[r].y);
        acc[r].x = fma(-x[r].y, v[u].y, acc[r].x);
        acc[r].y = fma(x[r].y, v[u].x, acc[r].y);
      }
  } else {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
#pragma unroll
      for (int r = 0; r < KX; ++r) {
        acc[r].x = fma(x[r].x, v[u].x, acc[r].x);
        acc[r].y = fma(x[r].x, v[u].y, acc[r].y);
      }
#pragma unroll
      for (int r = 0; r < KX; ++r) {
        acc[r].x = fma(-x[r].y, v[u].y, acc[r].x);
        acc[r].y = fma(x[r].y, v[u].x, acc[r].y);
      }
    }
  }
}

template <int KX, int MINB, int UNR, int ORD>
__global__ void __launch_bounds__(256, MINB) k(int reps, double2 *out) {
  constexpr int YT = 256;
  __shared__ double2 sY[8 * YT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *sW = sY + warp * YT;
  for (int i = lane; i < YT; i += 32) sW[i] = make_double2(1e-3 * i, -2e-3 * i);
  double2 x[KX], acc[KX];
  for (int r = 0; r < KX; ++r) {
    x[r] = make_double2(0.5 + lane * 1e-3 + r, 0.25 - r * 1e-3);
    acc[r] = make_double2(0.0, 0.0);
  }
  __syncwarp();
  for (int it = 0; it < reps; ++it)
    for (int y = 0; y + UNR - 1 < YT; y += UNR) {
      double2 v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) v[u] = sW[y + u];
      cfma<KX, UNR, ORD>(acc, x, v);
    }
  double2 s = make_double2(0, 0);
  for (int r = 0; r < KX; ++r) { s.x += acc[r].x; s.y += acc[r].y; }
  if (s.x == 1.2345) out[0] = s;
}

template <int KX, int MINB, int UNR, int ORD>
void run(const char *name, int nsm, double2 *out) {
  const int reps = 2000 * 8 / KX, grid = MINB * nsm;
  k<KX, MINB, UNR, ORD><<<grid, 256>>>(10, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<KX, MINB, UNR, ORD><<<grid, 256>>>(reps, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma = (double)grid * 256 * reps * 256 * KX * 4;
  printf("%-28s %.4e DFMA/s  (%s)\n", name, dfma / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double2 *out;
  cudaMalloc(&out, 16);
  run<8, 2, 4, 0>("KX8 2blk unr4 ord0 (kernel)", nsm, out);
  run<8, 2, 4, 1>("KX8 2blk unr4 ord1", nsm, out);
  run<8, 2, 2, 0>("KX8 2blk unr2 ord0", nsm, out);
  run<8, 3, 4, 0>("KX8 3blk unr4 ord0", nsm, out);
  run<8, 1, 4, 0>("KX8 1blk unr4 ord0", nsm, out);
  run<16, 1, 4, 0>("KX16 1blk unr4 ord0", nsm, out);
  run<16, 1, 2, 1>("KX16 1blk unr2 ord1", nsm, out);
  run<4, 3, 4, 0>("KX4 3blk unr4 ord0", nsm, out);
  run<4, 4, 8, 0>("KX4 4blk unr8 ord0", nsm, out);
  run<12, 1, 4, 0>("KX12 1blk unr4 ord0", nsm, out);
  return 0;
}
