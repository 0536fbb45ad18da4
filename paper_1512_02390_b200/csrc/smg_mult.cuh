// Multiplicative Schwarz sweep launcher (smg_mult.cu); handle in smg_abi.cu.
#pragma once
#include <cuda_runtime.h>

namespace smg {

constexpr int kMsMaxNP = 33;   // p <= 32

struct MsArgs {
  double* u;
  double* r;
  const double* Sx;     // m x m
  const double* Sy;
  const double* dinv;   // m x m
  const double* nu_bar; // (n_y, n_x) or nullptr
  const double* nu;     // diffusion: nodal nu (N_y, N_x), else nullptr
  // operator constants by value (kernel parameter space), row-major (p+1)^2
  double Ly[kMsMaxNP * kMsMaxNP];   // Poisson: stiff_y = (2/dy) L ; diffusion: D
  double Lx[kMsMaxNP * kMsMaxNP];   // Poisson: stiff_x ; diffusion: unused
  double my[kMsMaxNP], mx[kMsMaxNP];  // Poisson: mass_y, mass_x
  double w[kMsMaxNP];               // diffusion: GLL weights
  double cx, cy;        // diffusion: dy/dx, dx/dy
  int diffusion;
  int p, n_o, m, n_x, n_y, forward;
};

int mult_sweep_launch(const MsArgs& A, cudaStream_t st);

}  // namespace smg
