// Ascending half of the V-cycle in one launch (subsystem 3):
//
//   for l = 1..K:  u_l <- u_l + P_l u_{l-1}            (multigrid.py:247-248)
//
// with n_post = 0 (no smoothing between the prolongations, the reference's
// default cycle), on a chain of orders p_l = 2^l (p_K <= 16).  Every level
// shares the element mesh and the interpolation is element-local, so one warp
// per element carries the correction from the coarse level to level K
// without leaving registers / shared memory: at level l it forms the
// element's FULL (p_l+1)^2 node block, including the high-side nodes the
// neighbours own, as u_l[node] + (J C J^T)[node].
//
// Bitwise equal to the per-level prolongation (prolong_warp_kernel): the same
// fma chains in the same order (x pass over coarse columns from s = 0, then
// y pass over coarse rows from s = 0, then old + s), and a high-side node
// computed from this element's side equals the owner's value exactly -- the
// GLL end nodes coincide, so the J rows of the end nodes are one-hot and the
// shared edge depends only on the shared coarse edge (up to the sign of an
// exact zero).  Only u_K is written; u_1..u_{K-1} are read, not updated
// (nothing reads them after the cycle).
#include "smg_common.cuh"

namespace smg {

constexpr int kChainMaxK = 5;     // p_K <= 32
constexpr int kChainWarps = 8;

struct ChainArgs {
  const double* u0;                 // level 0 (p = 1) field (n_y, n_x)
  double* u[kChainMaxK + 1];        // u[1..K] level fields (u[K] updated in place)
  int n_x, n_y;
  // J_l: (2^l + 1) x (2^{l-1} + 1) row-major, levels 1..K, concatenated
  double J[3 * 2 + 5 * 3 + 9 * 5 + 17 * 9 + 33 * 17];
};

__host__ __device__ constexpr int chain_joff(int l) {
  // offset of J_l in ChainArgs::J
  int o = 0;
  for (int k = 1; k < l; ++k) o += ((1 << k) + 1) * ((1 << (k - 1)) + 1);
  return o;
}

// Old values of one level's element block (NB x NB from the element origin,
// high side wrapped) into O -- issued for every level before any compute, so
// the levels' global loads are in flight together.
template <int PF, bool FULL>
__device__ __forceinline__ void chain_fetch(const double* __restrict__ u, double* O, int ex, int ey, int n_x, int n_y,
                                            int lane) {
  constexpr int NB = FULL ? PF + 1 : PF;
  const int Nx = n_x * PF, Ny = n_y * PF;
  for (int o = lane; o < NB * NB; o += 32) {
    const int a = o / NB, b = o - a * NB;
    O[o] = u[(size_t)wrapi(ey * PF + a, Ny) * Nx + wrapi(ex * PF + b, Nx)];
  }
}

// One level: C (NC x NC, coarse element nodes incl. high side) -> F.
// FULL: F is (PF+1)^2 (intermediate level); else only the owned PF x PF nodes
// are formed and written straight to u (top level).  O: the fetched old values.
template <int PC, int PF, bool FULL>
__device__ __forceinline__ void chain_level(const double* __restrict__ J, const double* C, double* Tt, double* F,
                                            const double* O, double* __restrict__ u, int ex, int ey, int n_x,
                                            int lane) {
  constexpr int NC = PC + 1, NB = FULL ? PF + 1 : PF;
  const int Nx = n_x * PF;
  // x pass: Tt[ay][b] = sum_ax J[b][ax] C[ay][ax]   (b < NB)
  for (int o = lane; o < NC * NB; o += 32) {
    const int ay = o / NB, b = o - ay * NB;
    double s = 0.0;
#pragma unroll
    for (int ax = 0; ax < NC; ++ax) s = fma(J[b * NC + ax], C[ay * NC + ax], s);
    Tt[ay * NB + b] = s;
  }
  __syncwarp();
  // y pass: out[a][b] = old + sum_ay J[a][ay] Tt[ay][b]
  for (int o = lane; o < NB * NB; o += 32) {
    const int a = o / NB, b = o - a * NB;
    double s = 0.0;
#pragma unroll
    for (int ay = 0; ay < NC; ++ay) s = fma(J[a * NC + ay], Tt[ay * NB + b], s);
    const double v = O[o] + s;
    if (FULL) F[a * NB + b] = v;
    else u[(size_t)(ey * PF + a) * Nx + ex * PF + b] = v;
  }
  __syncwarp();
}

template <int K>
__global__ void __launch_bounds__(32 * kChainWarps) prolong_chain_kernel(const __grid_constant__ ChainArgs A) {
  SMG_PDL_ENTRY();
  constexpr int PK = 1 << K;
  constexpr int NMAX = (PK / 2 + 1) * (PK / 2 + 1) > 4 ? (PK / 2 + 1) * (PK / 2 + 1) : 4;   // largest C
  constexpr int TMAX = (PK / 2 + 1) * (PK + 1);                                               // largest Tt
  // old values of levels 1..K: (2^l + 1)^2 each below K, 2^K squared at K
  constexpr int OTOT = [] {
    int t = PK * PK;
    for (int l = 1; l < K; ++l) t += ((1 << l) + 1) * ((1 << l) + 1);
    return t;
  }();
  __shared__ double Cs[kChainWarps][2][NMAX];
  __shared__ double Ts[kChainWarps][TMAX];
  __shared__ double Os[kChainWarps][OTOT];
  // J rows are indexed per lane: from shared memory (the parameter bank
  // serializes divergent constant loads)
  constexpr int JTOT = chain_joff(K + 1);
  __shared__ double Js[JTOT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < JTOT; i += blockDim.x) Js[i] = A.J[i];
  __syncthreads();
  const int e = blockIdx.x * kChainWarps + warp;
  if (e >= A.n_x * A.n_y) return;
  const int ey = e / A.n_x, ex = e - ey * A.n_x;
  // level-0 element nodes (2 x 2, high side wrapped)
  if (lane < 4) {
    const int ay = lane >> 1, ax = lane & 1;
    Cs[warp][0][lane] = A.u0[(size_t)wrapi(ey + ay, A.n_y) * A.n_x + wrapi(ex + ax, A.n_x)];
  }
  double* Ow[kChainMaxK + 1];
  {
    int off = 0;
#pragma unroll
    for (int l = 1; l <= K; ++l) {
      Ow[l] = Os[warp] + off;
      off += l < K ? ((1 << l) + 1) * ((1 << l) + 1) : 0;
    }
  }
#define SMG_CHAIN_FETCH(L) \
  if constexpr (K >= L) chain_fetch<(1 << L), (L < K)>(A.u[L], Ow[L], ex, ey, A.n_x, A.n_y, lane);
  SMG_CHAIN_FETCH(1)
  SMG_CHAIN_FETCH(2)
  SMG_CHAIN_FETCH(3)
  SMG_CHAIN_FETCH(4)
  SMG_CHAIN_FETCH(5)
#undef SMG_CHAIN_FETCH
  __syncwarp();
  double* C = Cs[warp][0];
  double* F = Cs[warp][1];
#define SMG_CHAIN_LEVEL(L)                                                                                   \
  if constexpr (K >= L) {                                                                                    \
    if constexpr (L < K) {                                                                                   \
      chain_level<(1 << (L - 1)), (1 << L), true>(Js + chain_joff(L), C, Ts[warp], F, Ow[L], A.u[L], ex, ey, \
                                                  A.n_x, lane);                                              \
      double* t = C; C = F; F = t;                                                                           \
    } else {                                                                                                 \
      chain_level<(1 << (L - 1)), (1 << L), false>(Js + chain_joff(L), C, Ts[warp], F, Ow[L], A.u[L], ex, ey, \
                                                   A.n_x, lane);                                             \
    }                                                                                                        \
  }
  SMG_CHAIN_LEVEL(1)
  SMG_CHAIN_LEVEL(2)
  SMG_CHAIN_LEVEL(3)
  SMG_CHAIN_LEVEL(4)
  SMG_CHAIN_LEVEL(5)
#undef SMG_CHAIN_LEVEL
}

template <int K>
static int chain_launch(const ChainArgs& A, cudaStream_t st) {
  const int nel = A.n_x * A.n_y;
  launch(prolong_chain_kernel<K>, dim3((nel + kChainWarps - 1) / kChainWarps), dim3(32 * kChainWarps), 0, st, A);
  return check_launch("prolong_chain_kernel");
}

int prolong_chain_run(int K, int n_x, int n_y, const double* const* J, const double* u0, double* const* u,
                      cudaStream_t st) {
  if (K < 1 || K > 4) return SMG_EUNSUPPORTED;   // p_K <= 16 (one warp per element)
  ChainArgs A;
  A.u0 = u0;
  A.n_x = n_x;
  A.n_y = n_y;
  for (int l = 1; l <= K; ++l) {
    A.u[l] = u[l];
    const int n = ((1 << l) + 1) * ((1 << (l - 1)) + 1);
    for (int i = 0; i < n; ++i) A.J[chain_joff(l) + i] = J[l][i];
  }
  switch (K) {
    case 1: return chain_launch<1>(A, st);
    case 2: return chain_launch<2>(A, st);
    case 3: return chain_launch<3>(A, st);
    default: return chain_launch<4>(A, st);
  }
}

}  // namespace smg
