// The bottom of the V-cycle as ONE cooperative kernel ("V-cycle tail").
//
// Reference: v_cycle (multigrid.py:231-251) below the first level whose
// fields are large enough to fill the GPU.  At the BASELINE C2 mesh
// (64 x 64 elements) the levels p = 8, 4, 2 and the p = 1 coarse solve hold
// 262k, 65k, 16k and 4k DOFs: each of their ~16 kernels is a few hundred
// nanoseconds of work behind a launch + ramp + drain of several microseconds.
// Here they run as phases of one persistent grid (every CTA resident:
// cooperative launch), separated by grid barriers:
//
//   for l = K .. 1:                          (level l starts from u_l = 0)
//     A_l : FD solve of every element window of r = f_l (zero start:
//           A 0 = 0), W (.) S_y[(S_y^T B S_x) ./ (l_y (+) l_x)] S_x^T, into a
//           per-element buffer corr_l                    (schwarz.py:215-222)
//     BC_l: per tile of elements: u_l = sum of the window contributions
//           covering each node (mesh.py:142-150 scatter-add, in gather form),
//           r = f_l - A_l u_l (operators.py:49-54, 101-103), f_{l-1} = P^T r
//           on the tile's coarse nodes (multigrid.py:188-193, row-assigned P)
//   D   : T2 = Lp .* (Q_y^T f_0 Q_x)      (coarse pseudo-inverse, first half)
//   EF  : per tile of level-K elements: u_0 = Q_y T2 Q_x^T on the tile's
//         coarse nodes, then u_l += P u_{l-1} element by element up to level
//         K (multigrid.py:245-248); only u_K (and u_0) are written back.
//
// Every output node is written by exactly one thread, sums run in a fixed
// order: deterministic and bitwise reproducible.  The top level(s) stay on
// the tiled kernels.  Poisson operator, additive smoother with n_pre = 1,
// n_post = 0 on the tail levels, p <= 8, window m <= 17, coarse mesh <= 64^2.
#include <cooperative_groups.h>

#include "smg_common.cuh"
#include "smg_vtail.cuh"

namespace smg {

namespace cg = cooperative_groups;

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ int floordiv(int a, int b) {  // b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}
__device__ __forceinline__ int pmod(int a, int n) {
  int r = a % n;
  return r < 0 ? r + n : r;
}

// Copy n doubles into shared memory, dst[i] = *addr(i), with B independent
// L2 loads in flight per thread (every phase starts by staging its inputs:
// one dependent load chain per phase instead of one per element).
template <int B, typename AddrFn>
__device__ __forceinline__ void vt_stage(double* dst, int n, AddrFn addr) {
  for (int base = threadIdx.x; base < n; base += B * kVtThreads) {
    double v[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = base + k * kVtThreads;
      v[k] = i < n ? ldcg(addr(i)) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = base + k * kVtThreads;
      if (i < n) dst[i] = v[k];
    }
  }
}

__device__ __forceinline__ void vt_mark(const VtArgs* A, int k) {
  if (A->prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    A->prof[k] = (long long)t;
  }
}

// 2D variant: dst[r * ld + c] = *addr(r, c) for r < nr, c < nc; warp = row,
// lane = column, 4 x 2 loads in flight per thread.
template <typename AddrFn>
__device__ __forceinline__ void vt_stage2d(double* dst, int ld, int nr, int nc, AddrFn addr) {
  constexpr int NW = kVtThreads / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r0 = warp; r0 < nr; r0 += 4 * NW) {
    for (int c0 = lane; c0 < nc; c0 += 64) {
      double v[4][2];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r = r0 + k * NW, c = c0 + 32 * j;
          v[k][j] = (r < nr && c < nc) ? ldcg(addr(r, c)) : 0.0;
        }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r = r0 + k * NW, c = c0 + 32 * j;
          if (r < nr && c < nc) dst[r * ld + c] = v[k][j];
        }
    }
  }
}

// ---- A_l: FD window solves --------------------------------------------------
// A warp processes EPW = 32 / M elements at once; lane (slot, row) owns row
// `row` of element slot `slot` through the four contractions:
//   T1 = S_y^T B (row i: sum_k S_y[k][i] B[k][:]),  T2 = (T1 S_x) .* dinv,
//   T3 = S_y T2 (needs all rows: exchanged through shared memory),
//   out = W .* (T3 S_x^T)
template <int M>
__device__ __forceinline__ void vt_fd_phase(const VtLevel& L, int n_x, int n_y, double* sm) {
  constexpr int MM = M * M;
  constexpr int EPW = 32 / M;
  double* Sx = sm;
  double* Sy = Sx + MM;
  double* Dv = Sy + MM;
  double* Wy = Dv + MM;
  double* Wx = Wy + M;
  double* wbuf = Wx + M + 1;
  const int tid = threadIdx.x;
  for (int i = tid; i < MM; i += kVtThreads) {
    Sx[i] = L.Sx[i];
    Sy[i] = L.Sy[i];
    Dv[i] = L.dinv[i];
  }
  for (int i = tid; i < M; i += kVtThreads) {
    Wy[i] = L.wy[i];
    Wx[i] = L.wx[i];
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int slot = lane / M, row = lane - slot * M;
  double* B = wbuf + warp * (EPW * MM);
  const int p = L.p, n_o = L.n_o;
  const int N_x = n_x * p, N_y = n_y * p;
  const int n_el = n_x * n_y;
  const int nwarps = gridDim.x * (kVtThreads / 32);
  const double* __restrict__ f = L.f;
  for (int e0 = (blockIdx.x * (kVtThreads / 32) + warp) * EPW; e0 < n_el; e0 += nwarps * EPW) {
    {
      // window origins of the EPW elements (lane s < EPW computes element s)
      int rb = 0, cb = 0;
      if (lane < EPW && e0 + lane < n_el) {
        const int e = e0 + lane, ey = e / n_x, ex = e - ey * n_x;
        rb = ey * p - n_o;
        cb = ex * p - n_o;
      }
      constexpr int NL = (EPW * MM + 31) / 32;
      double tv[NL];
#pragma unroll
      for (int q = 0; q < NL; ++q) {
        const int idx = lane + 32 * q;
        const int s = idx / MM, r = idx - s * MM;
        const int k = r / M, c = r - k * M;
        const int ryb = __shfl_sync(0xffffffffu, rb, s < EPW ? s : 0);
        const int cxb = __shfl_sync(0xffffffffu, cb, s < EPW ? s : 0);
        tv[q] = 0.0;
        if (idx < EPW * MM && e0 + s < n_el)
          tv[q] = ldcg(f + (size_t)wrapi(ryb + k, N_y) * N_x + wrapi(cxb + c, N_x));
      }
#pragma unroll
      for (int q = 0; q < NL; ++q)
        if (lane + 32 * q < EPW * MM) B[lane + 32 * q] = tv[q];
    }
    __syncwarp();
    const int e = e0 + slot;
    const bool act = slot < EPW && e < n_el;
    double* Bs = B + (slot < EPW ? slot : 0) * MM;
    double t[M], v[M];
    if (act) {
#pragma unroll
      for (int j = 0; j < M; ++j) t[j] = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double s = Sy[k * M + row];
#pragma unroll
        for (int j = 0; j < M; ++j) t[j] = fma(s, Bs[k * M + j], t[j]);
      }
#pragma unroll
      for (int j = 0; j < M; ++j) v[j] = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
#pragma unroll
        for (int j = 0; j < M; ++j) v[j] = fma(t[k], Sx[k * M + j], v[j]);
      }
#pragma unroll
      for (int j = 0; j < M; ++j) v[j] *= Dv[row * M + j];
    }
    __syncwarp();
    if (act) {
#pragma unroll
      for (int j = 0; j < M; ++j) Bs[row * M + j] = v[j];
    }
    __syncwarp();
    if (act) {
#pragma unroll
      for (int j = 0; j < M; ++j) t[j] = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double s = Sy[row * M + k];
#pragma unroll
        for (int j = 0; j < M; ++j) t[j] = fma(s, Bs[k * M + j], t[j]);
      }
      double* out = L.corr + (size_t)e * MM + row * M;
      const double wy = Wy[row];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) s = fma(t[j], Sx[c * M + j], s);
        out[c] = s * (wy * Wx[c]);
      }
    }
    __syncwarp();
  }
}

// ---- BC_l: gather u, residual, restriction to level l-1 ----------------------
// One tile of te x te elements per CTA round.  All index arithmetic goes
// through per-row / per-column tables (the corr address of a window entry is
// separable: row part + column part), loops are (warp = row, lane = column).
template <int P, int PC, int NO>
__device__ __forceinline__ void vt_bc_phase(const VtArgs* A_, const VtLevel& L, const VtLevel& C, int n_x, int n_y, double* sm) {
  const int MB = 40 + 8 * (P == 8 ? 0 : (P == 4 ? 1 : 2));
  constexpr int p = P, pc = PC, n_o = NO, m = P + 1 + 2 * NO;
  constexpr int NP = p + 1, NC = pc + 1, mm = m * m;
  const int te = L.te;
  const int N_x = n_x * p, N_y = n_y * p, Nc_x = n_x * pc, Nc_y = n_y * pc;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kVtThreads / 32;
  const int RU = (te + 2) * p + 1, RR = (te + 1) * p;
  double* Lh = sm;                      // NP x NP
  double* Wa = Lh + NP * NP;            // p assembled weights
  double* Jm = Wa + p;                  // NP x NC
  double* U = Jm + NP * NC;             // RU x RU
  double* R = U + RU * RU;              // RR x RR
  double* H = R + RR * RR;              // RR x (te+1) x NC
  double* G = H + RR * (te + 1) * NC;   // (te+1)NC x (te+1)NC
  int* cntY = reinterpret_cast<int*>(G + (te + 1) * NC * (te + 1) * NC);
  int* cntX = cntY + RU;
  int* offY = cntX + RU;                // RU x 3 corr row offsets
  int* offX = offY + 3 * RU;            // RU x 3 corr column offsets
  int* rowG = offX + 3 * RU;            // RU: global row offset of U row (for u and f)
  int* colG = rowG + RU;                // RU: global column of U column
  for (int i = tid; i < NP * NP; i += kVtThreads) Lh[i] = L.L[i];
  for (int i = tid; i < p; i += kVtThreads) Wa[i] = L.wasm[i];
  for (int i = tid; i < NP * NC; i += kVtThreads) Jm[i] = L.J[i];
  const int tiles_x = (n_x + te - 1) / te, tiles_y = (n_y + te - 1) / te;
  const double* __restrict__ corr = L.corr;
  const double* __restrict__ f = L.f;
  const double cx = L.cx, cy = L.cy;
  for (int t = blockIdx.x; t < tiles_x * tiles_y; t += gridDim.x) {
    const int Ey = (t / tiles_x) * te, Ex = (t % tiles_x) * te;
    const int tey = min(te, n_y - Ey), tex = min(te, n_x - Ex);
    const int ruy = (tey + 2) * p + 1, rux = (tex + 2) * p + 1;
    const int rry = (tey + 1) * p, rrx = (tex + 1) * p;
    const int Y0 = (Ey - 2) * p, X0 = (Ex - 2) * p;
    __syncthreads();  // constants loaded / previous tile's smem reads done
    // index tables of the U region
    if (tid < ruy) {
      const int Y = Y0 + tid;
      const int e0 = floordiv(Y - n_o - 1, p), e1 = floordiv(Y + n_o, p);
      cntY[tid] = e1 - e0 + 1;
      for (int a = 0; a < 3; ++a) {
        const int e = e0 + a;
        offY[3 * tid + a] = (a <= e1 - e0) ? pmod(e, n_y) * n_x * mm + (Y - (e * p - n_o)) * m : 0;
      }
      rowG[tid] = pmod(Y, N_y) * N_x;
    } else if (tid >= 256 && tid < 256 + rux) {
      const int i = tid - 256, X = X0 + i;
      const int e0 = floordiv(X - n_o - 1, p), e1 = floordiv(X + n_o, p);
      cntX[i] = e1 - e0 + 1;
      for (int b = 0; b < 3; ++b) {
        const int e = e0 + b;
        offX[3 * i + b] = (b <= e1 - e0) ? pmod(e, n_x) * mm + (X - (e * p - n_o)) : 0;
      }
      colG[i] = pmod(X, N_x);
    }
    __syncthreads();
    vt_mark(A_, MB + 0);
    // (0) f on the residual region (U rows/cols p..) -> R, 8 loads in flight
    for (int ry0 = warp; ry0 < rry; ry0 += 4 * NW) {
      for (int rx0 = lane; rx0 < rrx; rx0 += 64) {
        double v[4][2];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int ry = ry0 + k * NW, rx = rx0 + 32 * j;
            v[k][j] = (ry < rry && rx < rrx) ? ldcg(f + rowG[ry + p] + colG[rx + p]) : 0.0;
          }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int ry = ry0 + k * NW, rx = rx0 + 32 * j;
            if (ry < rry && rx < rrx) R[ry * RR + rx] = v[k][j];
          }
      }
    }
    vt_mark(A_, MB + 1);
    // (1) u on the region: sum of the windows covering each node (<= CW per
    //     direction; ascending window rows, then columns: a fixed order).
    //     RB x 2 nodes per thread per round, all their loads in flight.
    {
      constexpr int CW = (2 * NO + 1 > P) ? 3 : 2;
      constexpr int RB = CW == 3 ? 2 : 4;
      for (int ry0 = warp; ry0 < ruy; ry0 += RB * NW) {
        for (int rx0 = lane; rx0 < rux; rx0 += 64) {
          double v[RB][2][CW * CW];
#pragma unroll
          for (int k = 0; k < RB; ++k) {
            const int ry = ry0 + k * NW;
            const bool iny = ry < ruy;
            const int cyn = iny ? cntY[ry] : 0;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int rx = rx0 + 32 * q;
              const bool in = iny && rx < rux;
              const int cxn = in ? cntX[rx] : 0;
#pragma unroll
              for (int a = 0; a < CW; ++a)
#pragma unroll
                for (int b = 0; b < CW; ++b)
                  v[k][q][a * CW + b] =
                      (in && a < cyn && b < cxn) ? ldcg(corr + offY[3 * ry + a] + offX[3 * rx + b]) : 0.0;
            }
          }
#pragma unroll
          for (int k = 0; k < RB; ++k) {
            const int ry = ry0 + k * NW;
            const bool owned_row = ry >= 2 * p && ry < (2 + tey) * p;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int rx = rx0 + 32 * q;
              if (ry < ruy && rx < rux) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < CW * CW; ++c) s += v[k][q][c];
                U[ry * RU + rx] = s;
                if (owned_row && rx >= 2 * p && rx < (2 + tex) * p) L.u[rowG[ry] + colG[rx]] = s;
              }
            }
          }
        }
      }
    }
    __syncthreads();
    vt_mark(A_, MB + 2);
    // (2) r = f - A u on the owned nodes of elements [E-1, E+te)
    for (int ry = warp; ry < rry; ry += NW) {
      const int a = ry % p;
      const int uy = ry + p;
      const double* urow = U + uy * RU;
      const double wya = cx * Wa[a];
      for (int rx = lane; rx < rrx; rx += 32) {
        const int b = rx % p;
        const int ux = rx + p;
        double sx = 0.0, sy = 0.0;
        for (int k = 0; k < NP; ++k) sx = fma(Lh[k * NP + b], urow[ux - b + k], sx);
        if (b == 0)
          for (int k = 0; k < NP; ++k) sx = fma(Lh[k * NP + p], urow[ux - p + k], sx);
        for (int k = 0; k < NP; ++k) sy = fma(Lh[k * NP + a], U[(uy - a + k) * RU + ux], sy);
        if (a == 0)
          for (int k = 0; k < NP; ++k) sy = fma(Lh[k * NP + p], U[(uy - p + k) * RU + ux], sy);
        R[ry * RR + rx] -= fma(wya, sx, cy * Wa[b] * sy);
      }
    }
    __syncthreads();
    vt_mark(A_, MB + 3);
    // (3) restriction, x pass: H[ry][exl][a] = sum_{b<p} R[ry][exl p + b] J[b][a]
    const int nex = tex + 1, ney = tey + 1;
    for (int ry = warp; ry < rry; ry += NW) {
      for (int q = lane; q < nex * NC; q += 32) {
        const int exl = q / NC, a = q - exl * NC;
        const double* rr = R + ry * RR + exl * p;
        double s = 0.0;
        for (int b = 0; b < p; ++b) s = fma(rr[b], Jm[b * NC + a], s);
        H[(ry * (te + 1) + exl) * NC + a] = s;
      }
    }
    __syncthreads();
    vt_mark(A_, MB + 4);
    //     y pass: G[eyl][ay][exl][ax] = sum_{b<p} J[b][ay] H[eyl p + b][exl][ax]
    const int GW = (te + 1) * NC;
    for (int gy = warp; gy < ney * NC; gy += NW) {
      const int eyl = gy / NC, ay = gy - eyl * NC;
      for (int gx = lane; gx < nex * NC; gx += 32) {
        const int exl = gx / NC, ax = gx - exl * NC;
        double s = 0.0;
        for (int b = 0; b < p; ++b) s = fma(Jm[b * NC + ay], H[(((eyl * p + b) * (te + 1)) + exl) * NC + ax], s);
        G[gy * GW + gx] = s;
      }
    }
    __syncthreads();
    vt_mark(A_, MB + 5);
    //     owned coarse nodes (elements Ey..Ey+tey-1 = eyl 1..tey, local a < pc)
    for (int cyy = warp; cyy < tey * pc; cyy += NW) {
      const int eyl = 1 + cyy / pc, ay = cyy - (eyl - 1) * pc;
      const size_t grow = (size_t)pmod(Ey * pc + cyy, Nc_y) * Nc_x;
      for (int cxx = lane; cxx < tex * pc; cxx += 32) {
        const int exl = 1 + cxx / pc, ax = cxx - (exl - 1) * pc;
        double s = G[(eyl * NC + ay) * GW + exl * NC + ax];
        if (ax == 0) s += G[(eyl * NC + ay) * GW + (exl - 1) * NC + pc];
        if (ay == 0) s += G[((eyl - 1) * NC + pc) * GW + exl * NC + ax];
        if (ax == 0 && ay == 0) s += G[((eyl - 1) * NC + pc) * GW + (exl - 1) * NC + pc];
        C.f[grow + pmod(Ex * pc + cxx, Nc_x)] = s;
      }
    }
  }
}

// ---- D: T2 = Lp .* (Q_y^T F Q_x), one row per CTA ------------------------------
__device__ void vt_pinv_rows(const VtArgs& A, double* sm) {
  const int nx = A.n_x, ny = A.n_y;
  const int tid = threadIdx.x;
  constexpr int KG = kVtThreads / kVtMaxN0;   // 8 partial-sum groups
  double* F = sm;                             // ny x nx
  double* QX = F + kVtMaxN0 * kVtMaxN0;       // nx x nx
  double* qc = QX + kVtMaxN0 * kVtMaxN0;      // column i of Q_y
  double* P = qc + kVtMaxN0;                  // KG x 64
  double* tv = P + KG * kVtMaxN0;             // 64
  const double* __restrict__ Fg = A.lv[0].f;
  const int x = tid % kVtMaxN0, kg = tid / kVtMaxN0;
  bool staged = false;
  for (int i = blockIdx.x; i < ny; i += gridDim.x) {
    __syncthreads();
    if (!staged) {
      vt_stage<8>(F, ny * nx, [&](int j) { return Fg + j; });
      vt_stage<8>(QX, nx * nx, [&](int j) { return A.Qx + j; });
      staged = true;
    }
    vt_stage<1>(qc, ny, [&](int k) { return A.Qy + (size_t)k * ny + i; });
    __syncthreads();
    double s = 0.0;
    if (x < nx)
      for (int k = kg; k < ny; k += KG) s = fma(qc[k], F[k * nx + x], s);
    P[kg * kVtMaxN0 + x] = s;
    __syncthreads();
    if (kg == 0) {
      double t = 0.0;
      for (int g = 0; g < KG; ++g) t += P[g * kVtMaxN0 + x];
      tv[x] = t;
    }
    __syncthreads();
    s = 0.0;
    if (x < nx)
      for (int j = kg; j < nx; j += KG) s = fma(tv[j], QX[j * nx + x], s);
    P[kg * kVtMaxN0 + x] = s;
    __syncthreads();
    if (kg == 0 && x < nx) {
      double t = 0.0;
      for (int g = 0; g < KG; ++g) t += P[g * kVtMaxN0 + x];
      A.T2[(size_t)i * nx + x] = t * A.Lp[(size_t)i * nx + x];
    }
  }
}

// ---- EF: coarse values on a level-K tile, prolongation chain up to level K ----
__device__ __forceinline__ double vt_dot(const double* __restrict__ a, const double* __restrict__ b, int sb, int n) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = 0;
  for (; k + 3 < n; k += 4) {
    s0 = fma(a[k], b[k * sb], s0);
    s1 = fma(a[k + 1], b[(k + 1) * sb], s1);
    s2 = fma(a[k + 2], b[(k + 2) * sb], s2);
    s3 = fma(a[k + 3], b[(k + 3) * sb], s3);
  }
  for (; k < n; ++k) s0 = fma(a[k], b[k * sb], s0);
  return (s0 + s1) + (s2 + s3);
}

// One level of the EF prolongation chain: level P (from P/2), region of the
// tile's nodes (with the high boundary unless this is the last level).
struct VtUpScratch {
  double* Jm;
  double* ub;
  int* rowG;
  int* colG;
  int* eT;
};

template <int P, int PK>
__device__ __forceinline__ void vt_up_level(const VtArgs& A, int l, double* vp, double* vc, int rwx, int Ey, int Ex,
                                            int tey, int tex, const VtUpScratch& S) {
  constexpr int p = P, pc = P / 2, NC = pc + 1;
  constexpr bool last = P == PK;
  constexpr int NW = kVtThreads / 32;
  constexpr int RMAX = kVtTE * kVtMaxP + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nx0 = A.n_x, ny0 = A.n_y;
  const VtLevel& L = A.lv[l];
  double* __restrict__ uL = L.u;
  const int N_x = nx0 * p, N_y = ny0 * p;
  const int ry_n = last ? tey * p : tey * p + 1, rx_n = last ? tex * p : tex * p + 1;
  double* Jm = S.Jm;
  double* ub = S.ub;
  int* rowG = S.rowG;
  int* colG = S.colG;
  int* eT = S.eT;
  __syncthreads();
  for (int i = tid; i < (p + 1) * NC; i += kVtThreads) Jm[i] = L.J[i];
  if (tid < ry_n) rowG[tid] = pmod(Ey * p + tid, N_y) * N_x;
  if (tid >= 128 && tid < 128 + rx_n) colG[tid - 128] = pmod(Ex * p + tid - 128, N_x);
  if (tid >= 256 && tid < 256 + RMAX) eT[tid - 256] = (tid - 256) / p;
  __syncthreads();
  for (int ry0 = warp; ry0 < ry_n; ry0 += 4 * NW) {
    for (int rx0 = lane; rx0 < rx_n; rx0 += 64) {
      double v[4][2];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int ry = ry0 + k * NW, rx = rx0 + 32 * j;
          v[k][j] = (ry < ry_n && rx < rx_n) ? ldcg(uL + rowG[ry] + colG[rx]) : 0.0;
        }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int ry = ry0 + k * NW, rx = rx0 + 32 * j;
          if (ry < ry_n && rx < rx_n) ub[ry * RMAX + rx] = v[k][j];
        }
    }
  }
  __syncthreads();
  vt_mark(&A, 20 + 2 * l);
  const int rwc = tex * p + 1;
  for (int ry = warp; ry < ry_n; ry += NW) {
    const int eyl = min(eT[ry], tey - 1), by = ry - eyl * p;
    double jy[NC];
#pragma unroll
    for (int ay = 0; ay < NC; ++ay) jy[ay] = Jm[by * NC + ay];
    for (int rx = lane; rx < rx_n; rx += 32) {
      const int exl = min(eT[rx], tex - 1), bx = rx - exl * p;
      const double* cb = vp + (eyl * pc) * rwx + exl * pc;
      double s = 0.0;
#pragma unroll
      for (int ay = 0; ay < NC; ++ay) {
        double sr = 0.0;
#pragma unroll
        for (int ax = 0; ax < NC; ++ax) sr = fma(Jm[bx * NC + ax], cb[ay * rwx + ax], sr);
        s = fma(jy[ay], sr, s);
      }
      const double val = ub[ry * RMAX + rx] + s;
      if (last) uL[rowG[ry] + colG[rx]] = val;
      else vc[ry * rwc + rx] = val;
    }
  }
  vt_mark(&A, 21 + 2 * l);
  if constexpr (!last) vt_up_level<2 * P, PK>(A, l + 1, vc, vp, rwc, Ey, Ex, tey, tex, S);
}

template <int PK>
__device__ __forceinline__ void vt_up_phase(const VtArgs& A, double* sm) {
  const int K = A.K, nx0 = A.n_x, ny0 = A.n_y;   // level 0 has p = 1: n_* nodes
  const int te = A.lv[K].te;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kVtThreads / 32;
  constexpr int RMAX = kVtTE * kVtMaxP + 1;
  constexpr int N0 = kVtMaxN0;
  constexpr int LD = N0 + 1;                       // padded row stride (no bank conflicts)
  double* T2 = sm;                                 // ny0 x nx0, stride LD
  double* QXr = T2 + N0 * LD;                      // (te+1) rows of Q_x
  double* QYr = QXr + (kVtTE + 1) * N0;            // (te+1) rows of Q_y
  double* V = QYr + (kVtTE + 1) * N0;              // (te+1) x ny0: V[c][i], stride LD
  double* Jm = V + LD * (kVtTE + 1);               // (p+1)(pc+1) of the current level
  double* va = Jm + (kVtMaxP + 1) * (kVtMaxP + 1);
  double* vb = va + RMAX * RMAX;
  double* ub = vb + RMAX * RMAX;                   // u_l on the tile region
  int* rowG = reinterpret_cast<int*>(ub + RMAX * RMAX);
  int* colG = rowG + RMAX;
  int* eT = colG + RMAX;                           // element of region index (clamped)
  VtUpScratch sm_lv{Jm, ub, rowG, colG, eT};
  const int tiles_x = (nx0 + te - 1) / te, tiles_y = (ny0 + te - 1) / te;
  bool staged = false;
  for (int t = blockIdx.x; t < tiles_x * tiles_y; t += gridDim.x) {
    const int Ey = (t / tiles_x) * te, Ex = (t % tiles_x) * te;
    const int tey = min(te, ny0 - Ey), tex = min(te, nx0 - Ex);
    __syncthreads();
    if (!staged) {
      vt_stage2d(T2, LD, ny0, nx0, [&](int r, int c) { return A.T2 + r * nx0 + c; });
      staged = true;
    }
    for (int c = warp; c < tex + 1; c += NW)
      for (int j = lane; j < nx0; j += 32) QXr[c * N0 + j] = A.Qx[(size_t)pmod(Ex + c, nx0) * nx0 + j];
    for (int r = warp; r < tey + 1; r += NW)
      for (int j = lane; j < ny0; j += 32) QYr[r * N0 + j] = A.Qy[(size_t)pmod(Ey + r, ny0) * ny0 + j];
    __syncthreads();
    vt_mark(&A, 16);
    // V[c][i] = sum_j T2[i][j] Q_x[X_c][j]
    for (int idx = tid; idx < ny0 * (tex + 1); idx += kVtThreads) {
      const int c = idx / ny0, i = idx - c * ny0;
      V[c * LD + i] = vt_dot(T2 + i * LD, QXr + c * N0, 1, nx0);
    }
    __syncthreads();
    vt_mark(&A, 17);
    // u0 on the (tey+1) x (tex+1) coarse nodes of the tile
    int rwx = tex + 1;
    for (int idx = tid; idx < (tey + 1) * rwx; idx += kVtThreads) {
      const int r = idx / rwx, c = idx - r * rwx;
      const double u0 = vt_dot(QYr + r * N0, V + c * LD, 1, ny0);
      va[idx] = u0;
      if (r < tey && c < tex) A.lv[0].u[(size_t)pmod(Ey + r, ny0) * nx0 + pmod(Ex + c, nx0)] = u0;
    }
    vt_up_level<2, PK>(A, 1, va, vb, tex + 1, Ey, Ex, tey, tex, sm_lv);
  }
}

template <int P>
__device__ __forceinline__ void vt_down(const VtArgs* A, int l, double* sm, cg::grid_group& grid, int& mk) {
  // level l has order P (= 2^l), one overlap layer: window m = P + 3
  vt_fd_phase<P + 3>(A->lv[l], A->n_x, A->n_y, sm);
  grid.sync();
  vt_mark(A, mk++);
  vt_bc_phase<P, P / 2, 1>(A, A->lv[l], A->lv[l - 1], A->n_x, A->n_y, sm);
  vt_mark(A, 40 + 8 * (P == 8 ? 0 : (P == 4 ? 1 : 2)) + 6);
  grid.sync();
  vt_mark(A, mk++);
  if constexpr (P > 2) vt_down<P / 2>(A, l - 1, sm, grid, mk);
}

// PK = order of the top tail level (levels 1..K have orders 2, 4, .., PK)
template <int PK>
__global__ void __launch_bounds__(kVtThreads, 1) vtail_kernel(const VtArgs* __restrict__ A) {
  extern __shared__ __align__(16) double smv[];
  cg::grid_group grid = cg::this_grid();
  int mk = 0;
  vt_mark(A, mk++);
  vt_down<PK>(A, A->K, smv, grid, mk);
  vt_pinv_rows(*A, smv);
  grid.sync();
  vt_mark(A, mk++);
  vt_up_phase<PK>(*A, smv);
  vt_mark(A, mk++);
}

using VtKernel = void (*)(const VtArgs*);
static VtKernel vt_kernel_for(int pk) {
  switch (pk) {
    case 2: return vtail_kernel<2>;
    case 4: return vtail_kernel<4>;
    case 8: return vtail_kernel<8>;
    default: return nullptr;
  }
}

size_t vtail_smem_bytes() {
  // FD phase: factors + per-warp windows (EPW * M * M <= 32 * M doubles), M <= 13
  constexpr size_t MX = 13;
  const size_t fd = 3 * MX * MX + 2 * MX + 1 + (kVtThreads / 32) * 32 * MX;
  // BC phase at te = kVtTE, p = kVtMaxP
  const size_t P = kVtMaxP, NP = P + 1, NC = P, te = kVtTE;
  const size_t RU = (te + 2) * P + 1, RR = (te + 1) * P;
  const size_t bc = NP * NP + P + NP * NC + RU * RU + RR * RR + RR * (te + 1) * NC +
                    (te + 1) * NC * (te + 1) * NC + (10 * RU + 8) / 2;
  const size_t RM = kVtTE * kVtMaxP + 1;
  const size_t up = kVtMaxN0 * (kVtMaxN0 + 1) + 3 * (kVtTE + 1) * (kVtMaxN0 + 1) + (kVtMaxP + 1) * (kVtMaxP + 1) + 3 * RM * RM +
                    (4 * RM + 8) / 2;
  const size_t d = 2 * kVtMaxN0 * kVtMaxN0 + (kVtThreads / kVtMaxN0 + 2) * kVtMaxN0;
  size_t mx = fd;
  if (bc > mx) mx = bc;
  if (up > mx) mx = up;
  if (d > mx) mx = d;
  return sizeof(double) * mx + 16;
}

int vtail_launch(const VtArgs* A_dev, int pk, int grid, cudaStream_t st) {
  VtKernel k = vt_kernel_for(pk);
  if (!k) { set_error("vtail: top tail order %d not compiled", pk); return SMG_EUNSUPPORTED; }
  const size_t smem = vtail_smem_bytes();
  static bool attr[3] = {false, false, false};
  const int slot = pk == 2 ? 0 : (pk == 4 ? 1 : 2);
  if (!attr[slot]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "vtail_kernel smem attribute");
    attr[slot] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kVtThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, A_dev);
  if (e != cudaSuccess) return cuda_fail(e, "vtail_kernel launch");
  return check_launch("vtail_kernel");
}

int vtail_grid() {
  static int g = 0;
  if (g == 0) {
    const size_t smem = vtail_smem_bytes();
    int dev = 0, sms = 0, per = 1 << 30;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (int pk : {2, 4, 8}) {
      VtKernel k = vt_kernel_for(pk);
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return -1;
      int q = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&q, k, kVtThreads, smem);
      if (e != cudaSuccess || q < 1) return -1;
      per = q < per ? q : per;
    }
    const int want = env_int("SMG_VTAIL_CTAS_PER_SM", 1);
    g = sms * (per < want ? per : want);
  }
  return g;
}

}  // namespace smg
