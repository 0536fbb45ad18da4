#pragma once
#include "smg_common.cuh"

namespace smg {

constexpr int kTrMaxP = 33;   // (p+1) bound
constexpr int kTrThreads = 256;

struct TrArgs {
  const double* __restrict__ src;
  double* __restrict__ dst;
  int pc, pf, n_x, n_y;
  int TX, TY, tiles_x, accumulate;
  double J[kTrMaxP * kTrMaxP];   // J[a*(pc+1)+ac], a in [0,pf], ac in [0,pc]
};

using TrFn = int (*)(const TrArgs&, int, bool, cudaStream_t);
TrFn transfer_dispatch(int pc, int pf);
size_t prolong_smem(int pc, int pf, int TX, int TY);
size_t restrict_smem(int pc, int pf, int TX, int TY);

}  // namespace smg
