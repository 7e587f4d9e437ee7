// grp.cuh -- a "cell group": the G lanes of one warp that integrate one cell.
//
// G = 1  : one cell per thread (n = 1..3: Nyx scalar, Robertson).
// G = 16 : one cell per half warp (n <= 16: H2/air, n = 10).
// G = 32 : one cell per warp (n <= 32: DRM19-class, n = 22).
//
// Component i of the cell is owned by lane (i mod G) as its r-th register
// slot, r = i / G (R = ceil(N/G) slots per lane).  Every scalar of the BDF
// state machine is replicated in all G lanes and computed identically, so
// control flow is uniform inside a group; lanes of *different* groups in the
// same warp may diverge (per-cell adaptive stepping with masked lanes).
//
// The WRMS reduction order is reading R15: lane l sums its own
// slots in increasing component order, then an xor butterfly with offsets
// G/2..1 -- the oracle emulates exactly this order.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bdfb {

template <int G_>
struct Grp {
  static constexpr int G = G_;
  static_assert(G == 1 || G == 2 || G == 4 || G == 8 || G == 16 || G == 32, "G must divide 32");
  int lane;        // lane inside the group, 0..G-1
  int wlane;       // lane inside the warp, 0..31
  int gbase;       // first warp lane of this group
  unsigned mask;   // warp-lane mask of the group

  __device__ __forceinline__ Grp() {
    wlane = threadIdx.x & 31;
    lane = (G == 1) ? 0 : (wlane & (G - 1));
    gbase = wlane - lane;
    mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  }

  __device__ __forceinline__ void sync() const {
    if (G > 1) __syncwarp(mask);
  }

  // sum over the group, xor butterfly (identical result in every lane)
  __device__ __forceinline__ double sum(double v) const {
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(mask, v, off, G));
    return v;
  }
  __device__ __forceinline__ double max(double v) const {
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) v = fmax(v, __shfl_xor_sync(mask, v, off, G));
    return v;
  }
  __device__ __forceinline__ int imax(int v) const {
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) v = ::max(v, __shfl_xor_sync(mask, v, off, G));
    return v;
  }
  __device__ __forceinline__ int ior(int v) const {
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) v |= __shfl_xor_sync(mask, v, off, G);
    return v;
  }
  // value of v in group lane src
  __device__ __forceinline__ double bcast(double v, int src) const {
    return (G == 1) ? v : __shfl_sync(mask, v, src, G);
  }
  __device__ __forceinline__ int bcast(int v, int src) const {
    return (G == 1) ? v : __shfl_sync(mask, v, src, G);
  }
};

// Component bookkeeping for a system of size N owned by a group of G lanes.
template <int N_, int G_>
struct Layout {
  static constexpr int N = N_;
  static constexpr int G = G_;
  static constexpr int R = (N + G - 1) / G;   // register slots per lane
  __device__ __forceinline__ static int comp(int lane, int r) { return lane + G * r; }
  __device__ __forceinline__ static bool valid(int lane, int r) { return lane + G * r < N; }
};

}  // namespace bdfb
