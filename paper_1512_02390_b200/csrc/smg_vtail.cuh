// V-cycle tail: the lower levels of a V-cycle as one cooperative kernel
// (smg_vtail.cu).  Host-side handle in smg_abi.cu (smg_vtail_*).
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace smg {

constexpr int kVtMaxLevels = 4;   // tail levels 1..K, K <= 4
constexpr int kVtMaxP = 8;
constexpr int kVtMaxM = 13;      // compiled window sizes: 5, 6, 7, 8, 9, 11, 13
constexpr int kVtTE = 6;          // max tile edge in elements (BC / EF phases)
constexpr int kVtMaxN0 = 64;      // coarse mesh <= 64 x 64
constexpr int kVtThreads = 512;

struct VtLevel {
  int p, n_o, m, te;
  double cx, cy;                  // dy/dx, dx/dy
  const double* Sx;               // m x m, S[k][i]
  const double* Sy;
  const double* dinv;             // m x m, 1/(lam_y[i] + lam_x[j])
  const double* wx;               // m
  const double* wy;               // m
  const double* L;                // (p+1)^2 reference stiffness L-hat
  const double* wasm;             // p assembled GLL weights
  const double* J;                // (p+1) x (p_{l-1}+1) interpolation from level l-1
  double* f;
  double* u;
  double* corr;                   // n_el x m x m window solves
};

struct VtArgs {
  int K, n_x, n_y;                // tail levels 1..K; element mesh
  VtLevel lv[kVtMaxLevels + 1];   // lv[0]: coarse p = 1 (f, u only)
  const double* Qx;               // coarse pseudo-inverse factors
  const double* Qy;
  const double* Lp;
  double* T2;                     // n_y x n_x workspace
  long long* prof;                // nullable: globaltimer at phase boundaries (CTA 0)
};

size_t vtail_smem_bytes();
int vtail_grid();                 // CTAs of the cooperative grid (<= 0: unavailable)
int vtail_launch(const VtArgs* A_dev, int pk, int grid, cudaStream_t st);  // A_dev: device copy; pk: top tail order

}  // namespace smg
