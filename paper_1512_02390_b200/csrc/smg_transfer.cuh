#pragma once
#include "smg_common.cuh"

namespace smg {

constexpr int kTrMaxP = 33;   // (p+1) bound

struct TrArgs {
  const double* __restrict__ src;
  double* __restrict__ dst;
  int n_x, n_y, tiles_x, accumulate;
  int bulk;                 // 1: bulk row copies (even row lengths, 16-byte aligned fields)
  double J[kTrMaxP * 17];   // J[a*(pc+1)+ac], a in [0,pf], ac in [0,pc]
};

using TrFn = int (*)(const TrArgs&, int n_x, int n_y, bool prolong, cudaStream_t);
// launcher for (p_c, p_f) on an n_x x n_y mesh (largest compiled tile that divides it)
TrFn transfer_dispatch(int pc, int pf);

// Halo-free restriction (smg_rw.cu): warp per fine element + ring workspace of
// n_x n_y (2 p_c + 1) doubles + fixup launch; nullptr where it is not compiled.
using RwFn = int (*)(const TrArgs&, double* ring, cudaStream_t);
RwFn rw_dispatch(int pc, int pf);
int rw_fixup(int pc, double* dst, const double* ring, int n_x, int n_y, cudaStream_t st);
// Warp-per-fine-element prolongation (smg_rw.cu); nullptr where it is not compiled.
using PrwFn = int (*)(const TrArgs&, cudaStream_t);
PrwFn prw_dispatch(int pc, int pf);

}  // namespace smg
