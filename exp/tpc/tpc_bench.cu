// experiment: thread-per-cell straight-line RHS vs the warp-cooperative RHS (same physics)
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2405_01713_b200/csrc/gen/tpc_drm19_class.cuh"
using namespace bdfb;
__global__ void __launch_bounds__(128) k_tpc(long long N, const double* y, const double* rho, double* f, int reps) {
  long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= N) return;
  double yy[22], ff[22];
  for (int k = 0; k < 22; ++k) yy[k] = y[k * N + c];
  double r = rho[c];
  for (int it = 0; it < reps; ++it) {
    tpc_rhs_drm19_class(yy, r, ff);
    yy[0] += 1e-300 * ff[0];   // keep a dependence
  }
  for (int k = 0; k < 22; ++k) f[k * N + c] = ff[k];
}
int main() {
  long long N = 1 << 20; int reps = 20;
  double *y, *rho, *f;
  cudaMalloc(&y, N * 22 * 8); cudaMalloc(&rho, N * 8); cudaMalloc(&f, N * 22 * 8);
  // plausible state: Y = 1/21, T = 1500, rho = 2.4e-4
  double* h = (double*)malloc(N * 22 * 8);
  for (long long c = 0; c < N; ++c) { for (int k = 0; k < 21; ++k) h[k * N + c] = 1.0 / 21; h[21 * N + c] = 1200 + (c % 1000); }
  cudaMemcpy(y, h, N * 22 * 8, cudaMemcpyHostToDevice);
  for (long long c = 0; c < N; ++c) h[c] = 2.4e-4;
  cudaMemcpy(rho, h, N * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_tpc<<<(N + 127) / 128, 128>>>(N, y, rho, f, 1);
  cudaEventRecord(a);
  k_tpc<<<(N + 127) / 128, 128>>>(N, y, rho, f, reps);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("thread-per-cell RHS: %.3f ms for %lld x %d RHS -> %.3e RHS/s\n", ms, N, reps, N * reps / (ms * 1e-3));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
