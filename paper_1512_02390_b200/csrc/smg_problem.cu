// Device-side problem generation: nodal coordinates,
// the diffusivity field, manufactured loads and exact-solution samples of
// operators.py:110-199, evaluated per node on the GPU instead of on the host
// (at C5 one field is 151 M DOF = 1.2 GB: host evaluation + H2D dominated the
// setup).  Same expressions in the same order as the reference; the only
// difference is the FP64 sin/cos implementation (<= 2 ulp).
#include <vector>

#include "smg_common.cuh"

namespace smg {

struct ProbConsts {
  double loc[33];   // (xi_b + 1) / 2, b in [0, p)
  double wq[33];    // assembled GLL weight of local node b: w_b (+ w_p for b = 0)
  double w0, wp;    // w_0, w_p (node b = 0 adds the previous element's w_p)
};

__device__ __forceinline__ double pi_d() { return 3.141592653589793; }

// kind: 0 nu = 1 + nu_hat sin(2pi(x-s)) sin(2pi(y-s))      (operators.py:167-173)
//       1 Poisson load  W(y) W(x) * 2 pi^2 sin(pi x) sin(pi y)  (:143-164, before project_mean)
//       2 diffusion load W(y) W(x) * -(nu lap u + grad nu.grad u), u = sin 2pi x sin 2pi y (:176-199)
//       3 Poisson exact samples   sin(pi x) sin(pi y)
//       4 diffusion exact samples sin(2pi x) sin(2pi y)
__global__ void __launch_bounds__(256) problem_field_kernel(int kind, int p, int n_x, int n_y, double dx, double dy,
                                                            const __grid_constant__ ProbConsts C, double nu_hat,
                                                            double s, double* __restrict__ out) {
  SMG_PDL_ENTRY();
  const int N_x = n_x * p, N_y = n_y * p;
  const long n = (long)N_x * N_y;
  for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (long)gridDim.x * blockDim.x) {
    const int Y = (int)(idx / N_x), X = (int)(idx - (long)Y * N_x);
    const int ex = X / p, bx = X - ex * p, ey = Y / p, by = Y - ey * p;
    const double x = (ex + C.loc[bx]) * dx, y = (ey + C.loc[by]) * dy;
    const double pi = pi_d(), tp = 2.0 * pi;
    double v;
    if (kind == 0) {
      v = 1.0 + nu_hat * sin(tp * (x - s)) * sin(tp * (y - s));
    } else if (kind == 3) {
      v = sin(pi * x) * sin(pi * y);
    } else if (kind == 4) {
      v = sin(tp * x) * sin(tp * y);
    } else {
      // assembled quadrature: (d/2) w_b, plus (d/2) w_p of the previous element at b = 0
      const double hx = dx / 2.0, hy = dy / 2.0;
      const double wx = bx == 0 ? hx * C.w0 + hx * C.wp : hx * C.wq[bx];
      const double wy = by == 0 ? hy * C.w0 + hy * C.wp : hy * C.wq[by];
      double src;
      if (kind == 1) {
        src = 2.0 * (pi * pi) * (sin(pi * x) * sin(pi * y));
      } else {
        const double u = sin(tp * x) * sin(tp * y);
        const double ux = tp * cos(tp * x) * sin(tp * y);
        const double uy = tp * sin(tp * x) * cos(tp * y);
        const double lap = -2.0 * (tp * tp) * u;
        const double nv = 1.0 + nu_hat * sin(tp * (x - s)) * sin(tp * (y - s));
        const double nx = tp * nu_hat * cos(tp * (x - s)) * sin(tp * (y - s));
        const double ny = tp * nu_hat * sin(tp * (x - s)) * cos(tp * (y - s));
        src = -(nv * lap + nx * ux + ny * uy);
      }
      v = (wy * wx) * src;
    }
    out[idx] = v;
  }
}

// Quadrature-weighted element mean of a nodal field (operators.py:94-98):
// out[ey][ex] = sum_ij nu[ey p + i][ex p + j] w_i w_j / 4 (periodic).
__global__ void __launch_bounds__(256) element_mean_kernel(int p, int n_x, int n_y, const __grid_constant__ ProbConsts C,
                                                           const double* __restrict__ nu, double* __restrict__ out) {
  SMG_PDL_ENTRY();
  const int N_x = n_x * p, N_y = n_y * p;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_x * n_y) return;
  const int ey = e / n_x, ex = e - ey * n_x;
  double acc = 0.0;
  for (int i = 0; i <= p; ++i) {
    const double* row = nu + (size_t)((ey * p + i) % N_y) * N_x;
    const double wi = i == p ? C.wp : (i == 0 ? C.w0 : C.wq[i]);
    double r = 0.0;
    for (int j = 0; j <= p; ++j) {
      const double wj = j == p ? C.wp : (j == 0 ? C.w0 : C.wq[j]);
      r = fma(row[(ex * p + j) % N_x], wi * wj, r);
    }
    acc += r;
  }
  out[e] = acc / 4.0;
}

static ProbConsts make_consts(int p, const double* nodes, const double* weights) {
  ProbConsts C;
  for (int b = 0; b < 33; ++b) { C.loc[b] = 0.0; C.wq[b] = 0.0; }
  for (int b = 0; b < p; ++b) {
    C.loc[b] = (nodes[b] + 1.0) / 2.0;
    C.wq[b] = weights[b];
  }
  C.w0 = weights[0];
  C.wp = weights[p];
  return C;
}

}  // namespace smg

using namespace smg;

extern "C" int smg_problem_field(int kind, int p, int n_x, int n_y, double dx, double dy, const double* nodes,
                                 const double* weights, double nu_hat, double shift, double* out, void* stream) {
  if (kind < 0 || kind > 4 || p < 1 || p > 32 || n_x < 1 || n_y < 1 || !nodes || !weights || !out) {
    set_error("smg_problem_field: bad argument");
    return SMG_EINVAL;
  }
  const ProbConsts C = make_consts(p, nodes, weights);
  const long n = (long)n_x * p * n_y * p;
  const long blocks = (n + 255) / 256;
  launch(problem_field_kernel, dim3((unsigned)(blocks < 148 * 16 ? blocks : 148 * 16)), dim3(256), 0,
         as_stream(stream), kind, p, n_x, n_y, dx, dy, C, nu_hat, shift, out);
  return check_launch("problem_field_kernel");
}

extern "C" int smg_element_mean(int p, int n_x, int n_y, const double* weights, const double* nu, double* out,
                                void* stream) {
  if (p < 1 || p > 32 || n_x < 1 || n_y < 1 || !weights || !nu || !out) {
    set_error("smg_element_mean: bad argument");
    return SMG_EINVAL;
  }
  std::vector<double> dummy(p + 1, 0.0);
  const ProbConsts C = make_consts(p, dummy.data(), weights);
  const int ne = n_x * n_y;
  launch(element_mean_kernel, dim3((ne + 255) / 256), dim3(256), 0, as_stream(stream), p, n_x, n_y, C, nu, out);
  return check_launch("element_mean_kernel");
}
