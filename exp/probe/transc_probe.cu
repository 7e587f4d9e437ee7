// transc_probe.cu -- FP64-pipe cost of the transcendentals in the generated RHS/J
// (fexp of csrc/fexp.cuh, libdevice log, log10, exp).  One kernel per function,
// each evaluating it once per element; ncu's executed DFMA/DADD/DMUL counts per
// element give the algorithmic flop weight bench.py charges per call
// ("each exp/log weighted by its FP64-pipe instruction count,
// measured once on the box").  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -fmad=false -I../../paper_2405_01713_b200/csrc transc_probe.cu -o transc_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "fexp.cuh"

#define PROBE(NAME, EXPR)                                                                         \
  __global__ void probe_##NAME(const double* __restrict__ in, double* __restrict__ out, int n) { \
    const int i = blockIdx.x * blockDim.x + threadIdx.x;                                          \
    if (i < n) {                                                                                  \
      const double x = in[i];                                                                     \
      out[i] = (EXPR);                                                                            \
    }                                                                                             \
  }
PROBE(copy, x)
PROBE(fexp, bdfb::fexp(x))
PROBE(log, log(x))
PROBE(log10, log10(x))
PROBE(exp, exp(x))

int main() {
  const int n = 1 << 24;
  double *in, *out;
  cudaMalloc(&in, n * sizeof(double));
  cudaMalloc(&out, n * sizeof(double));
  double* h = new double[n];
  for (int i = 0; i < n; ++i) h[i] = 0.5 + 30.0 * (double)i / n;   // positive: valid for log and exp
  cudaMemcpy(in, h, n * sizeof(double), cudaMemcpyHostToDevice);
  const int b = 256, g = (n + b - 1) / b;
  probe_copy<<<g, b>>>(in, out, n);
  probe_fexp<<<g, b>>>(in, out, n);
  probe_log<<<g, b>>>(in, out, n);
  probe_log10<<<g, b>>>(in, out, n);
  probe_exp<<<g, b>>>(in, out, n);
  cudaDeviceSynchronize();
  printf("elements %d\n", n);
  return 0;
}
