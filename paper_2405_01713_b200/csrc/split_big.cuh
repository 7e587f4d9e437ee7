// split_big.cuh -- the setup kernels of the SPLIT per-cell integrator for mechanisms larger than a warp
// (n > 32: the 53-species GRI-3.0-class mechanism of config C5, n = 54), B200 / sm_100a.
//
// The thread-per-cell control (K_ctl) and RHS (K_rhs, the generated straight-line RHS) are the SPLIT kernels
// of bdf_split.cuh, unchanged; only the matrix setup changes with n:
//   K_jac (split_jac_lanes_kernel): one cell per warp, the table-driven analytic Jacobian of the lanes model
//     (mech_lanes.cuh: lane l owns rows l + 32 r) written straight into the slot's column-major J record;
//   K_lu (split_lu_rows_kernel): M = I - gamma J and its LU with partial pivoting, one cell per 64 threads
//     holding the rows in registers, six cells per 384-thread block in lockstep (glu_columns of
//     global_lanes.cuh: the listing's LU_FACTOR operation for operation, reading R16), factors written in the
//     SPLIT LU record layout (column-major in pivoted row order | 1/U_kk | perm) that K_ctl's Newton solve reads.
// The group-model slot of the SPLIT templates (GM) is a stub for these mechanisms: the THREAD kernel's
// cooperative stages that use it are not instantiated.
#pragma once
#include "bdf_split.cuh"
#include "gen/mech_gri53_class.cuh"
#include "gen/tpc_gri53_class.cuh"
#include "global_lanes.cuh"
#include "mech_lanes.cuh"

namespace bdfb {

// stand-in for the group model of the SPLIT templates when n > 32
template <int NN>
struct GMStub {
  static constexpr int N = NN, G = 64, SG = 0, JG = 0;
};

template <class Mech>
struct LanesOf;
template <>
struct LanesOf<Tpc_gri53_class> {
  using type = ModelMechR<mech_gri53_class::Traits, 32>;
  using GM = GMStub<Tpc_gri53_class::N>;
};

// K_jac, one cell per warp (grid-stride over the Jacobian list), two warps per block; the Jacobian is assembled in
// shared memory (its sparse scattered row updates are read-modify-writes: in the J record they were HBM round
// trips) and copied to the record coalesced; status -> TS.coop
constexpr int JL_WARPS = 2;
template <class Mech>
struct JacLanesSmem {
  using MR = typename LanesOf<Mech>::type;
  static constexpr int MS = Mech::N | 1;
  static constexpr int PER_WARP = Mech::N * MS + MR::SG + MR::JG;   // doubles
};
template <class Mech, class GM, int LS>
__global__ void __launch_bounds__(32 * JL_WARPS) split_jac_lanes_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  using MR = typename LanesOf<Mech>::type;
  constexpr int N = Mech::N, R = MR::R, MS = JacLanesSmem<Mech>::MS;
  extern __shared__ double smem[];
  Grp<32> g;
  double* A = smem + (threadIdx.x >> 5) * JacLanesSmem<Mech>::PER_WARP;
  double* sc = A + N * MS;
  const long long cnt = b.cnt[3 * (it & 1) + 1], warps = (long long)gridDim.x * JL_WARPS;
  for (long long e = ((long long)blockIdx.x * 32 * JL_WARPS + threadIdx.x) >> 5; e < cnt; e += warps) {
    const long long slot = b.jlist[e];
    const typename SP::W w = SP::ws(b, slot);
    TS* t = SP::ts(b, slot);
    double yy[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = g.lane + 32 * r;
      yy[r] = i < N ? w.yq(i) : 0.0;
    }
    // row i, column j at A[j MS + i], then to the record's column-major J[j N + i]
    const int rv = MR::jac(g, yy, t->aux, A, 1, MS, sc, sc + MR::SG);
    g.sync();
    if (!rv) {
      double* J = b.J + slot * SP::JREC;
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int i = g.lane + 32 * r;
          if (i < N) J[j * N + i] = A[j * MS + i];
        }
    }
    if (g.lane == 0) t->coop = rv ? 1 : 0;
    g.sync();
  }
}

// K_lu, six cells per block (grid-stride over the setup list in block-uniform trips)
// K_lu block shape for n > 32: two 192-thread blocks per SM (3 cells each; GLUShared is sized for gl_lu's 6)
// instead of gl_lu's one 384-thread block: a block waiting at its per-column barriers no longer idles the SM
// (C5P K_lu 929 -> 846 ms, profiles/r2/history.md)
template <int NN>
struct LUR {
  static constexpr int TC = GLU<NN>::TC, CPB = 192 / TC > 0 ? 192 / TC : 1, T = CPB * TC, BPS = 384 / T > 0 ? 384 / T : 1;
  static_assert(CPB <= GLU<NN>::CPB, "GLUShared holds GLU<NN>::CPB cells");
};
template <class Mech, class GM, int LS>
__global__ void __launch_bounds__(LUR<Mech::N>::T, LUR<Mech::N>::BPS) split_lu_rows_kernel(SplitBufs b, int it) {
  using SP = Split<Mech, GM, LS>;
  constexpr int N = Mech::N, TC = LUR<N>::TC, CPB = LUR<N>::CPB;
  __shared__ GLUShared<N> sh;
  const int cb = threadIdx.x / TC, i = threadIdx.x % TC;
  const long long cnt = b.cnt[3 * (it & 1)];
  for (long long e0 = (long long)blockIdx.x * CPB; e0 < cnt; e0 += (long long)gridDim.x * CPB) {
    const long long e = e0 + cb;
    bool alive = e < cnt;
    const long long slot = alive ? b.slist[e] : 0;
    TS* t = SP::ts(b, slot);
    if (alive && t->coop) alive = false;     // the Jacobian failed: the resumed trip handles it (uniform per cell)
    const double gm = alive ? t->gamma : 0.0;
    const double* J = b.J + slot * SP::JREC;
    const bool own = i < N && alive;
    double a[N];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = own ? (i == j ? 1.0 : 0.0) - gm * J[j * N + i] : 0.0;
    int pos = i;
    double dinv = 0.0;
    const int info = glu_columns<N>(sh, a, pos, dinv, i, cb, alive, std::make_integer_sequence<int, N>{});
    if (alive && !info && own) {
      double* lu = SP::lurec(b, slot);
#pragma unroll
      for (int j = 0; j < N; ++j) lu[(j * N + pos) * LU_STRIDE] = a[j];
      lu[(SP::LU_INVD + pos) * LU_STRIDE] = dinv;
      if (LU_STRIDE == 1) reinterpret_cast<int*>(lu + SP::LU_PERM)[pos] = i;
      else lu[(SP::LU_PERM + pos) * LU_STRIDE] = (double)i;
    }
    if (alive && i == 0) t->coop = info;
  }
}

}  // namespace bdfb
