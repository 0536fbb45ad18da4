// C ABI of libsmg: handle construction, validation and dispatch.
// See include/smg.h for the contract and the reference call site each entry
// point replaces.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "smg_common.cuh"
#include "smg_fd.cuh"
#include "smg_fdt.cuh"
#include "smg_op.cuh"
#include "smg_transfer.cuh"
#include "smg_rr.cuh"
#include "smg_mult.cuh"

namespace smg {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int env_int(const char* name, int def) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : def;
}

bool sync_check_enabled() {
  static const bool on = [] {
    const char* s = getenv("SMG_SYNC_CHECK");
    return s && s[0] == '1';
  }();
  return on;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SMG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return SMG_ECUDA;
}

int ccg_update(double* x, double* r, const double* p, const double* q, int64_t n, double* S, int ro,
               int rn, double tol, int it, double* ws, cudaStream_t st);
int ccg_direction(double* p, const double* r, int64_t n, const double* S, int ro, int rn, cudaStream_t st);
int ccg_dot(const double* x, const double* y, int64_t n, double* out, const double* S, double* ws, cudaStream_t st);
int pcg_update(double* x, double* r, const double* p, const double* q, int64_t n, double* S, int ro, double tol,
               int it, double* ws, cudaStream_t st);
int pcg_scale(double* z, int64_t n, double scale, const double* S, cudaStream_t st);
int pcg_coop(int nx, int ny, double dx, double dy, const double* tab, const double* nu, double* x, double* r,
             double* p0, double* p1, double* z, double* W, double* part, double* S, double tol, int max_iter,
             cudaStream_t st);
int pcg_dscale(const double* in, double* out, const double* nu, int64_t n, const double* S, cudaStream_t st);
int pinv_fft(int nx, int ny, double dx, double dy, const double* f, double* u, double* ws, const double* tab,
             cudaStream_t st);
std::vector<double> fft_table(int nx, int ny);
int pinv_cluster(int nx, int ny, const double* Qx, const double* QxT, const double* Qy, const double* Lp,
                 const double* f, double* u, cudaStream_t st);
int pinv_small(int nx, int ny, const double* Qx, const double* Qy, const double* Lp, const double* f,
               double* tmp, double* u, cudaStream_t st);
int gemm(int M, int N, int K, const double* A, int lda, int tA, const double* B, int ldb, int tB,
         double* C, int ldc, const double* S, cudaStream_t st);


}  // namespace smg

using namespace smg;

// ---------------------------------------------------------------------------
struct smg_op {
  int kind, p, n_x, n_y;
  smg::OpLaunchFn fn;
  double dx, dy;
  std::vector<double> Mt, w, wasm;
  const double* nu;
  // norm partials (one per CTA) live in the caller's workspace (smg_op_ws_doubles)
  int n_ctas;
  double* dfrag = nullptr;   // DMMA operand fragments (smg_opd.cu): diffusion p = 24, Poisson p = 32
};

struct smg_schwarz {
  int p, n_o, n_x, n_y, m;
  std::vector<double> Sx, Sy, wx, wy;
  double* dinv;
  const double* inv_nu;
  struct Cls { int start, stride, count; };
  std::vector<Cls> cx, cy;
  // tiled even/odd path (smg_fdt.cuh); tiled == false -> coloured dense path
  bool tiled;
  smg::FDTLaunchFn fdt;
  int TX, TY, ntx, nty;
  std::vector<double> Sye, Syo, Sxe, Sxo;
  double* dinv_perm;
  size_t ws_doubles;  // ring workspace the caller passes to correct / smooth
  bool eo_dmma;   // even/odd DMMA stages inside the TMA-pipelined tiled kernel
  bool pair;      // paired-line kernel (smg_fdp.cuh)
};

struct smg_transfer {
  int pc, pf, n_x, n_y;
  std::vector<double> J;
  smg::TrFn fn;
  smg::RwFn rw;   // halo-free restriction (smg_rw.cu) or nullptr
  bool rr_opw = false;   // (8, 16): residual + restriction in the warp-per-element operator kernel needs the ring too
  smg::PrwFn prw; // warp-per-fine-element prolongation (smg_rw.cu) or nullptr
};

struct smg_coarse {
  int n_x, n_y;
  double dx, dy;
  double* Qx;   // n_x x n_x
  double* QxT;  // its transpose
  double* Qy;   // n_y x n_y
  double* Lp;   // n_y x n_x pseudo-inverse eigenvalues
  double* fft = nullptr;   // FFT path table (smg_fft.cu fft_table), power-of-two meshes
};

namespace smg {
int ccg_cta_run(int nx, int ny, double cx, double cy, const double* f0, double* u0, double tol, int max_iter,
                double* S, cudaStream_t st);
int prolong_chain_run(int K, int n_x, int n_y, const double* const* J, const double* u0, double* const* u,
                      cudaStream_t st);
}

namespace {

// tools/time_fd1.py on B200 (us, DFMA vs even/odd DMMA): 256^2 p=16 230 / 286,
// p=24 585 / 593, 128^2 p=32 401 / 372 -> DMMA from m = 35 (p = 32) up
bool fd_prefers_eo_dmma(int m) { return m >= 33; }

// Split S (m x m, row-major S[k][i]) into symmetrized even/odd halves.
// Returns false if some eigenvector is not (numerically) even or odd.
bool even_odd_split(const double* S, int m, std::vector<double>& Se, std::vector<double>& So,
                    std::vector<int>& perm) {
  const int HE = (m + 1) / 2, HO = m / 2;
  double smax = 0.0;
  for (int i = 0; i < m * m; ++i) smax = std::fmax(smax, std::fabs(S[i]));
  std::vector<int> ev, od;
  for (int i = 0; i < m; ++i) {
    double dot = 0.0, asym_e = 0.0, asym_o = 0.0;
    for (int k = 0; k < m; ++k) {
      dot += S[k * m + i] * S[(m - 1 - k) * m + i];
      asym_e = std::fmax(asym_e, std::fabs(S[k * m + i] - S[(m - 1 - k) * m + i]));
      asym_o = std::fmax(asym_o, std::fabs(S[k * m + i] + S[(m - 1 - k) * m + i]));
    }
    const bool is_even = dot > 0.0;
    if ((is_even ? asym_e : asym_o) > 1e-6 * smax) return false;
    (is_even ? ev : od).push_back(i);
  }
  if ((int)ev.size() != HE || (int)od.size() != HO) return false;
  Se.assign((size_t)HE * HE, 0.0);
  So.assign((size_t)HO * HO + 1, 0.0);
  for (int k = 0; k < HE; ++k)
    for (int a = 0; a < HE; ++a)
      Se[k * HE + a] = 0.5 * (S[k * m + ev[a]] + S[(m - 1 - k) * m + ev[a]]);
  for (int k = 0; k < HO; ++k)
    for (int a = 0; a < HO; ++a)
      So[k * HO + a] = 0.5 * (S[k * m + od[a]] - S[(m - 1 - k) * m + od[a]]);
  perm = ev;
  perm.insert(perm.end(), od.begin(), od.end());
  return true;
}

}  // namespace

namespace smg {
// Profiling aid for the tiled Schwarz kernel: per-phase clock64 sums of
// thread 0 of every CTA, enabled by SMG_FDT_PHASES=1 (else nullptr: no cost).
unsigned long long* fdt_phase_buffer() {
  static unsigned long long* buf = nullptr;
  static const int on = env_int("SMG_FDT_PHASES", 0);
  if (on && buf == nullptr && cudaMalloc(&buf, sizeof(unsigned long long) * FDT_NPH) == cudaSuccess)
    cudaMemset(buf, 0, sizeof(unsigned long long) * FDT_NPH);
  return buf;
}
}  // namespace smg

extern "C" {

const char* smg_last_error(void) { return g_err; }

int smg_debug_fdt_phases(unsigned long long* out, int n) {
  unsigned long long* buf = smg::fdt_phase_buffer();
  if (buf == nullptr) return set_error("smg_debug_fdt_phases: SMG_FDT_PHASES=1 not set"), SMG_EINVAL;
  const int k = n < smg::FDT_NPH ? n : smg::FDT_NPH;
  cudaError_t e = cudaMemcpy(out, buf, sizeof(unsigned long long) * k, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(buf, 0, sizeof(unsigned long long) * smg::FDT_NPH);
  return e == cudaSuccess ? SMG_OK : cuda_fail(e, "smg_debug_fdt_phases");
}
int smg_version(void) { return 1; }
int64_t smg_launch_count(void) { return g_launches.load(); }

int smg_device_ok(void) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_error("no CUDA device: %s", e != cudaSuccess ? cudaGetErrorString(e) : "count=0");
    return 0;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) {
    set_error("libsmg is built for sm_100a; device has compute capability major %d", major);
    return 0;
  }
  return 1;
}

// ---- operators --------------------------------------------------------------
int smg_op_create(smg_op_t** h, int kind, int p, int n_x, int n_y, double dx, double dy,
                  const double* weights, const double* mat, const double* nu_dev) {
  if (!h || !weights || !mat || p < 1 || n_x < 2 || n_y < 2 || !(dx > 0) || !(dy > 0) ||
      (kind != 0 && kind != 1) || (kind == 1 && !nu_dev)) {
    set_error("smg_op_create: bad argument");
    return SMG_EINVAL;
  }
  int ctas = 0;
  OpLaunchFn fn = op_dispatch(p, kind == 1, n_x, n_y, &ctas);
  if (!fn) {
    set_error("smg_op_create: order p=%d not compiled in", p);
    return SMG_EUNSUPPORTED;
  }
  smg_op* o = new (std::nothrow) smg_op();
  if (!o) return SMG_ENOMEM;
  o->kind = kind; o->p = p; o->n_x = n_x; o->n_y = n_y; o->dx = dx; o->dy = dy;
  o->Mt.assign(mat, mat + (p + 1) * (p + 1));
  o->w.assign(weights, weights + p + 1);
  o->wasm.resize(p);
  for (int a = 0; a < p; ++a) o->wasm[a] = weights[a];
  o->wasm[0] = weights[0] + weights[p];
  o->nu = nu_dev;
  o->fn = fn;
  o->n_ctas = ctas;
  cudaError_t e = cudaSuccess;
  // The tensor-core path builds its fragments from averaged halves of `mat`:
  // exact only if L-hat is centro-symmetric (Poisson) or D anti-centro-
  // symmetric (diffusion), as the reference's GLL matrices are.  Any other
  // matrix keeps the CUDA-core kernels (dfrag stays null -> opd_launch declines).
  bool sym_ok = true;
  {
    const int NP = p + 1;
    double mmax = 0.0, dev = 0.0;
    for (int i = 0; i < NP * NP; ++i) mmax = std::fmax(mmax, std::fabs(mat[i]));
    for (int i = 0; i < NP; ++i)
      for (int j = 0; j < NP; ++j) {
        const double a = mat[i * NP + j], b = mat[(p - i) * NP + (p - j)];
        dev = std::fmax(dev, std::fabs(kind == 1 ? a + b : a - b));
      }
    sym_ok = dev <= 1e-14 * (mmax > 0.0 ? mmax : 1.0);
    // the diffusion fragments carry w[n] for both G[n] and G[P-n]
    if (kind == 1)
      for (int i = 0; i < NP; ++i)
        if (std::fabs(weights[i] - weights[p - i]) > 1e-14 * std::fabs(weights[i])) sym_ok = false;
  }
  if (sym_ok && opd_applies(p, kind == 1)) {
    std::vector<double> fr;
    opd_fragments(p, kind == 1, mat, weights, fr);
    e = cudaMalloc(&o->dfrag, sizeof(double) * fr.size());
    if (e == cudaSuccess) e = cudaMemcpy(o->dfrag, fr.data(), sizeof(double) * fr.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { delete o; return cuda_fail(e, "smg_op_create"); }
  }
  *h = o;
  return SMG_OK;
}

int smg_op_destroy(smg_op_t* h) {
  if (!h) return SMG_OK;
  if (h->dfrag) cudaFree(h->dfrag);
  delete h;
  return SMG_OK;
}

static int op_run(const smg_op_t* h, const double* u, const double* f, double* out, double* partials,
                  cudaStream_t st, double* ring = nullptr) {
  const bool norm = partials != nullptr;
  OpLaunch L;
  L.u = u; L.f = f; L.out = out; L.nu = h->nu; L.partials = partials;
  L.ring = ring;
  L.p = h->p; L.n_x = h->n_x; L.n_y = h->n_y; L.diffusion = h->kind;
  L.cx = h->dy / h->dx; L.cy = h->dx / h->dy;
  L.Mt = h->Mt.data(); L.w = h->w.data(); L.wasm = h->wasm.data();
  if (!norm) {
    int rc = (h->kind == 0 && ring != nullptr) ? opl_launch(L, st) : 1;
    if (rc == 1) rc = opd_launch(L, h->dfrag, st);
    if (rc == 1 && h->kind == 0) rc = opw_launch(L, st);
    if (rc != 1) return rc;
  }
  return h->fn(L, st);
}

int smg_op_residual(const smg_op_t* h, const double* u, const double* f, double* out, void* stream) {
  if (!h || !u || !out || u == out) { set_error("smg_op_residual: bad argument"); return SMG_EINVAL; }
  return op_run(h, u, f, out, nullptr, as_stream(stream));
}

size_t smg_op_ring_doubles(const smg_op_t* h) {
  return (h && h->dfrag && opd_applies(h->p, h->kind != 0)) ? (size_t)h->n_x * h->n_y * 2 * h->p : 0;
}

int smg_op_residual_ws(const smg_op_t* h, const double* u, const double* f, double* out, double* ring,
                       void* stream) {
  if (!h || !u || !out || u == out) { set_error("smg_op_residual_ws: bad argument"); return SMG_EINVAL; }
  return op_run(h, u, f, out, nullptr, as_stream(stream), smg_op_ring_doubles(h) ? ring : nullptr);
}

int smg_sum_partials(const double* part, int nb, double* out, void* stream);

size_t smg_op_ws_doubles(const smg_op_t* h) {
  // per-CTA norm partials of the generic kernel, then the reduction workspace of the dot pass
  return h ? (size_t)h->n_ctas + smg_reduce_ws_doubles() : 0;
}

int smg_op_residual_norm2(const smg_op_t* h, const double* u, const double* f, double* out,
                          double* norm2_out, double* ws, void* stream) {
  if (!h || !u || !out || u == out || !norm2_out || !ws) {
    set_error("smg_op_residual_norm2: bad argument");
    return SMG_EINVAL;
  }
  int rc = op_run(h, u, f, out, ws, as_stream(stream));
  if (rc) return rc;
  return smg_sum_partials(ws, h->n_ctas, norm2_out, stream);
}

int smg_op_apply_dot(const smg_op_t* h, const double* u, double* out, double* dot_out, double* ws, double* ring,
                     void* stream) {
  if (!h || !u || !out || u == out || !dot_out || !ws) {
    set_error("smg_op_apply_dot: bad argument");
    return SMG_EINVAL;
  }
  const long ndof = (long)h->n_x * h->n_y * h->p * h->p;
  static const int fused = env_int("SMG_APPLY_DOT", 1);
  if (fused && h->kind == 0 && (h->p == 8 || h->p == 16) && h->n_x % 2 == 0 && h->n_y % 2 == 0 &&
      (long)(h->n_x / 2) * (h->n_y / 2) <= (long)h->n_ctas + (long)smg_reduce_ws_doubles()) {
    OpLaunch L;
    L.u = u; L.f = nullptr; L.out = out; L.nu = h->nu; L.partials = nullptr;
    L.p = h->p; L.n_x = h->n_x; L.n_y = h->n_y; L.diffusion = h->kind;
    L.cx = h->dy / h->dx; L.cy = h->dx / h->dy;
    L.Mt = h->Mt.data(); L.w = h->w.data(); L.wasm = h->wasm.data();
    int nct = 0;
    const int rc = opw_apply_dot(L, ws, &nct, as_stream(stream));
    if (rc == 0) return smg_sum_partials(ws, nct, dot_out, stream);
    if (rc != 1) return rc;
  }
  if (fused && h->kind == 1 && h->p == 24 && h->dfrag && ring && smg_op_ring_doubles(h) && h->nu) {
    // tensor-core diffusion kernel: the product accumulated per persistent CTA (at most
    // 148 x 6 partials, behind the generic kernel's)
    OpLaunch L;
    L.u = u; L.f = nullptr; L.out = out; L.nu = h->nu; L.partials = nullptr;
    L.p = h->p; L.n_x = h->n_x; L.n_y = h->n_y; L.diffusion = h->kind;
    L.cx = h->dy / h->dx; L.cy = h->dx / h->dy;
    L.Mt = h->Mt.data(); L.w = h->w.data(); L.wasm = h->wasm.data();
    int nct = 0;
    double* part = ws + h->n_ctas;
    const int rc = opdh_apply_dot(L, h->dfrag, ring, part, &nct, as_stream(stream));
    if (rc == 0) return smg_sum_partials(part, nct, dot_out, stream);
    if (rc != 1) return rc;
  }
  int rc = op_run(h, u, nullptr, out, nullptr, as_stream(stream), smg_op_ring_doubles(h) ? ring : nullptr);
  if (rc) return rc;
  double* red = ws + h->n_ctas;
  cudaError_t e = cudaMemsetAsync(red, 0, sizeof(double) * smg_reduce_ws_doubles(), as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "smg_op_apply_dot");
  return smg_dot(u, out, (int64_t)ndof, dot_out, red, stream);
}

int smg_op_residual_norm2_ws(const smg_op_t* h, const double* u, const double* f, double* out,
                             double* norm2_out, double* ws, double* ring, void* stream) {
  if (!h || !u || !out || u == out || !norm2_out || !ws) {
    set_error("smg_op_residual_norm2_ws: bad argument");
    return SMG_EINVAL;
  }
  // specialised residual kernel + dot pass where that is the faster pair (B200: C3 p = 32
  // 301 -> 165 us, C4 p = 16 160 -> 123 us; equal at C2, which keeps the fused partials)
  const long ndof = (long)h->n_x * h->n_y * h->p * h->p;
  const bool tensor = ring != nullptr && smg_op_ring_doubles(h) > 0;
  const bool warp = h->kind == 0 && (h->p == 8 || h->p == 16) && ndof >= (1L << 22);
  static const int mode = env_int("SMG_NORM_DOT", 1);
  if (!mode || !(tensor || warp)) return smg_op_residual_norm2(h, u, f, out, norm2_out, ws, stream);
  int rc = op_run(h, u, f, out, nullptr, as_stream(stream), ring);
  if (rc) return rc;
  // the dot's reduction workspace sits behind the generic kernel's partials; its arrival
  // counter must start at zero (the kernel resets it after use): cleared here, so the
  // caller's buffer needs no initialisation
  double* red = ws + h->n_ctas;
  cudaError_t e = cudaMemsetAsync(red, 0, sizeof(double) * smg_reduce_ws_doubles(), as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "smg_op_residual_norm2_ws");
  return smg_dot(out, out, (int64_t)ndof, norm2_out, red, stream);
}

// ---- additive Schwarz ---------------------------------------------------------
static void colour_classes(int n, int c, std::vector<smg_schwarz::Cls>& out) {
  // c = colours needed so that same-colour windows are disjoint; if n is not
  // a multiple of c, the trailing n % c elements get a class each.
  const int full = (n / c) * c;
  for (int k = 0; k < c && k < full; ++k) out.push_back({k, c, full / c});
  for (int e = full; e < n; ++e) out.push_back({e, 1, 1});
}

int smg_schwarz_destroy(smg_schwarz_t* h);

int smg_schwarz_create(smg_schwarz_t** h, int p, int n_o, int n_x, int n_y, const double* S_x,
                       const double* S_y, const double* lam_x, const double* lam_y,
                       const double* w_x, const double* w_y, const double* inv_nu_dev) {
  if (!h || !S_x || !S_y || !lam_x || !lam_y || !w_x || !w_y || p < 1 || n_o < 0 || n_o > p - 1 ||
      n_x < 2 || n_y < 2) {
    set_error("smg_schwarz_create: bad argument");
    return SMG_EINVAL;
  }
  const int m = p + 1 + 2 * n_o;
  if (m > p * n_x || m > p * n_y) {
    set_error("subdomain window (%d nodes) wraps onto itself on a %dx%d mesh at p=%d; reduce n_o", m, n_x, n_y, p);
    return SMG_EINVAL;
  }
  if (!fd_dispatch(m)) {
    set_error("smg_schwarz_create: window size m=%d not compiled in", m);
    return SMG_EUNSUPPORTED;
  }
  smg_schwarz* s = new (std::nothrow) smg_schwarz();
  if (!s) return SMG_ENOMEM;
  s->p = p; s->n_o = n_o; s->n_x = n_x; s->n_y = n_y; s->m = m;
  s->Sx.assign(S_x, S_x + m * m);
  s->Sy.assign(S_y, S_y + m * m);
  s->wx.assign(w_x, w_x + m);
  s->wy.assign(w_y, w_y + m);
  s->inv_nu = inv_nu_dev;
  std::vector<double> dinv(m * m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) dinv[i * m + j] = 1.0 / (lam_y[i] + lam_x[j]);
  cudaError_t e = cudaMalloc(&s->dinv, sizeof(double) * m * m);
  if (e == cudaSuccess) e = cudaMemcpy(s->dinv, dinv.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { delete s; return cuda_fail(e, "smg_schwarz_create"); }
  // colours per direction: windows of elements c apart are disjoint iff (c-1) p > 2 n_o
  int c = 2;
  while ((c - 1) * p <= 2 * n_o) ++c;
  colour_classes(n_x, c > n_x ? n_x : c, s->cx);
  colour_classes(n_y, c > n_y ? n_y : c, s->cy);
  // tiled even/odd path
  s->tiled = false;
  s->dinv_perm = nullptr; s->ws_doubles = 0;
  std::vector<int> px, py;
  const char* force = getenv("SMG_FD_DENSE");
  s->fdt = nullptr;
  // contraction engine: even/odd FP64 tensor cores (DMMA) or CUDA-core DFMA;
  // SMG_FD_ENGINE=dmma_eo|dfma overrides the per-m default
  const char* eng = getenv("SMG_FD_ENGINE");
  s->eo_dmma = eng ? (std::strcmp(eng, "dmma_eo") == 0) : fd_prefers_eo_dmma(m);
  // the tiled kernel folds the weights into its synthesis factors, which needs
  // mirror-symmetric weights (true for every reference weight kind, to 1 ulp)
  double wasym = 0.0, wmax = 0.0;
  for (int k = 0; k < m; ++k) {
    wasym = std::fmax(wasym, std::fmax(std::fabs(w_x[k] - w_x[m - 1 - k]), std::fabs(w_y[k] - w_y[m - 1 - k])));
    wmax = std::fmax(wmax, std::fmax(std::fabs(w_x[k]), std::fabs(w_y[k])));
  }
  const bool w_sym = wasym <= 1e-14 * (wmax > 0.0 ? wmax : 1.0);
  const bool eo_ok = w_sym && even_odd_split(S_x, m, s->Sxe, s->Sxo, px) &&
                     even_odd_split(S_y, m, s->Sye, s->Syo, py);
  // the paired-line kernel (smg_fdp.cuh) where it is compiled, unless
  // SMG_FD_ENGINE names one of the fdt_kernel engines
  const bool want_pair = !eng || std::strcmp(eng, "pair") == 0;
  s->pair = false;
  if (!(force && force[0] == '1') && eo_ok && want_pair) {
    s->fdt = fdp_dispatch(p, n_o, n_x, n_y, &s->TX, &s->TY);
    s->pair = s->fdt != nullptr;
  }
  if (!(force && force[0] == '1') && eo_ok &&
      (s->fdt != nullptr || (s->fdt = fdt_dispatch(p, n_o, n_x, n_y, &s->TX, &s->TY, s->eo_dmma)) != nullptr)) {
    s->ntx = n_x / s->TX; s->nty = n_y / s->TY;
    const int nt = s->ntx * s->nty;
    const size_t RX = (size_t)s->TX * p + 2 * n_o + 1, RY = (size_t)s->TY * p + 2 * n_o + 1;
    std::vector<double> dp((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) dp[i * m + j] = 1.0 / (lam_y[py[i]] + lam_x[px[j]]);
    e = cudaMalloc(&s->dinv_perm, sizeof(double) * m * m);
    if (e == cudaSuccess) e = cudaMemcpy(s->dinv_perm, dp.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice);
    s->ws_doubles = (size_t)nt * (RX * RY - (size_t)s->TX * p * s->TY * p);  // ring nodes per tile
    if (e != cudaSuccess) { smg_schwarz_destroy(s); return cuda_fail(e, "smg_schwarz_create (tiles)"); }
    s->tiled = true;
  }
  *h = s;
  return SMG_OK;
}

int smg_schwarz_destroy(smg_schwarz_t* h) {
  if (!h) return SMG_OK;
  cudaFree(h->dinv);
  if (h->dinv_perm) cudaFree(h->dinv_perm);
  delete h;
  return SMG_OK;
}

static FDLaunch fd_base(const smg_schwarz_t* h) {
  FDLaunch L;
  std::memset(&L, 0, sizeof(L));
  L.inv_nu = h->inv_nu; L.dinv = h->dinv;
  L.p = h->p; L.n_o = h->n_o; L.N_x = h->p * h->n_x; L.N_y = h->p * h->n_y; L.n_x = h->n_x;
  L.Sx = h->Sx.data(); L.Sy = h->Sy.data(); L.wx = h->wx.data(); L.wy = h->wy.data();
  L.apply_weight = 1;
  return L;
}

size_t smg_schwarz_ws_doubles(const smg_schwarz_t* h) { return h ? h->ws_doubles : 0; }

int smg_schwarz_info(const smg_schwarz_t* h, int* engine, int* tx, int* ty) {
  if (!h) return set_error("smg_schwarz_info: null handle"), SMG_EINVAL;
  if (engine) {
    int tx0 = 0, ty0 = 0;
    const bool dm = h->tiled && !h->pair && h->eo_dmma &&
                    h->fdt != fdt_dispatch(h->p, h->n_o, h->n_x, h->n_y, &tx0, &ty0, false);
    *engine = !h->tiled ? 0 : h->pair ? 3 : dm ? 2 : 1;
  }
  if (tx) *tx = h->tiled ? h->TX : 0;
  if (ty) *ty = h->tiled ? h->TY : 0;
  return SMG_OK;
}

static int schwarz_correct(const smg_schwarz_t* h, const double* r, double* u, double* ws, int u_zero,
                           void* stream) {
  if (h->tiled) {
    FDTLaunch T;
    T.r = r; T.u = u; T.u_zero = u_zero;
    T.inv_nu = h->inv_nu; T.dinv = h->dinv_perm; T.ws = ws;
    T.N_x = h->p * h->n_x; T.N_y = h->p * h->n_y; T.n_x = h->n_x; T.ntx = h->ntx; T.nty = h->nty;
    T.Sye = h->Sye.data(); T.Syo = h->Syo.data(); T.Sxe = h->Sxe.data(); T.Sxo = h->Sxo.data();
    T.wx = h->wx.data(); T.wy = h->wy.data();
    const int rc = h->fdt(T, as_stream(stream));
    if (rc != SMG_EUNSUPPORTED) return rc;
    // TMA cannot describe these buffers (odd row length or unaligned base):
    // the coloured dense kernel below computes the same correction
  }
  if (u_zero) {
    cudaError_t e = cudaMemsetAsync(u, 0, sizeof(double) * h->p * h->n_x * h->p * h->n_y, as_stream(stream));
    if (e != cudaSuccess) return cuda_fail(e, "schwarz_correct");
  }
  FDLaunchFn fn = fd_dispatch(h->m);
  FDLaunch L = fd_base(h);
  L.src = r; L.dst = u;
  for (const auto& cy : h->cy)
    for (const auto& cx : h->cx) {
      L.x0 = cx.start; L.xs = cx.stride; L.xc = cx.count;
      L.y0 = cy.start; L.ys = cy.stride; L.yc = cy.count;
      int rc = fn(L, as_stream(stream));
      if (rc) return rc;
    }
  return SMG_OK;
}

int smg_schwarz_correct(const smg_schwarz_t* h, const double* r, double* u, double* ws, void* stream) {
  if (!h || !r || !u || r == u || (h->ws_doubles && !ws)) {
    set_error("smg_schwarz_correct: bad argument");
    return SMG_EINVAL;
  }
  return schwarz_correct(h, r, u, ws, 0, stream);
}

int smg_schwarz_smooth(const smg_schwarz_t* h, const smg_op_t* op, double* u, const double* f,
                       double* work, double* ws, int n_it, int u_is_zero, void* stream) {
  return smg_schwarz_smooth_ws(h, op, u, f, work, ws, nullptr, n_it, u_is_zero, stream);
}

int smg_schwarz_smooth_ws(const smg_schwarz_t* h, const smg_op_t* op, double* u, const double* f,
                          double* work, double* ws, double* op_ring, int n_it, int u_is_zero, void* stream) {
  if (!h || !op || !u || !f || !work || n_it < 0 || op->p != h->p || op->n_x != h->n_x || op->n_y != h->n_y ||
      (h->ws_doubles && !ws)) {
    set_error("smg_schwarz_smooth: bad argument");
    return SMG_EINVAL;
  }
  for (int it = 0; it < n_it; ++it) {
    const double* r = f;
    if (!(it == 0 && u_is_zero)) {
      int rc = smg_op_residual_ws(op, u, f, work, op_ring, stream);
      if (rc) return rc;
      r = work;
    }
    int rc = schwarz_correct(h, r, u, ws, (it == 0 && u_is_zero) ? 1 : 0, stream);
    if (rc) return rc;
  }
  return SMG_OK;
}

int smg_fd_solve_blocks(const smg_schwarz_t* h, const double* blocks, double* out, int nb,
                        int apply_weight, void* stream) {
  if (!h || !blocks || !out || nb < 0) { set_error("smg_fd_solve_blocks: bad argument"); return SMG_EINVAL; }
  FDLaunch L = fd_base(h);
  L.src = blocks; L.dst = out; L.inv_nu = nullptr; L.blocks_mode = 1; L.nb = nb;
  L.apply_weight = apply_weight;
  L.xc = 1; L.yc = 1;
  return fd_dispatch(h->m)(L, as_stream(stream));
}

// ---- transfers --------------------------------------------------------------
int smg_transfer_create(smg_transfer_t** h, int p_c, int p_f, int n_x, int n_y, const double* J) {
  if (!h || !J || p_c < 1 || p_f <= p_c || n_x < 2 || n_y < 2) {
    set_error("smg_transfer_create: bad argument");
    return SMG_EINVAL;
  }
  TrFn fn = transfer_dispatch(p_c, p_f);
  if (!fn) { set_error("smg_transfer_create: (p_c,p_f)=(%d,%d) not compiled in", p_c, p_f); return SMG_EUNSUPPORTED; }
  smg_transfer* t = new (std::nothrow) smg_transfer();
  if (!t) return SMG_ENOMEM;
  t->pc = p_c; t->pf = p_f; t->n_x = n_x; t->n_y = n_y; t->fn = fn;
  // SMG_RW=0 keeps the tiled kernels (B200, us per restriction, tiled -> halo-free: C3 p_f = 32
  // 176 -> 77; 256^2 p_f = 24 208 -> 157, p_f = 16 110 -> 69; C2 15.4 -> 13.3)
  const int rw_mode = env_int("SMG_RW", 1);   // read per handle (create time only)
  // p_f = 16 on small meshes (C2): the extra fixup launch costs more inside the V-cycle's
  // dependent chain than the kernel gains (C2 V-cycle 105.2 -> 107.8 us with it)
  const bool big = p_f >= 24 || (long)n_x * n_y >= 16384 || rw_mode == 2;
  t->rw = (rw_mode && big) ? rw_dispatch(p_c, p_f) : nullptr;
  // (8, 16) and (4, 8): residual + restriction inside the warp-per-element operator kernel
  // (smg_opw.cu; the ring below is its workspace) -- C4 (256^2 elements) pair 159 -> 135 us at
  // p_f = 16, 74 -> 36 us at p_f = 8; C2 (64^2) V-cycle in the replayed graph 103.6 -> 100.3 us
  // with both.  SMG_RR_OPW = 0: residual kernel + restriction kernel (or rr_kernel at p_f <= 8)
  // (2, 4) as well: four elements per warp (C4 level-4 pair 21.5 -> 12.5 us; C2's replayed
  // V-cycle 99.87 -> 99.67 us, i.e. even)
  t->rr_opw = env_int("SMG_RR_OPW", 1) != 0 &&
              ((p_c == 8 && p_f == 16) || (p_c == 4 && p_f == 8) || (p_c == 2 && p_f == 4));
  // SMG_PRW: 0 never, 1 where measured faster, 2 wherever compiled (B200, tools/time_prolong.py,
  // us tiled -> warp per fine element: C3 p_f = 32 95.3 -> 79.9; 256^2 p_f = 24 156.7 -> 162.9,
  // p_f = 16 76.9 -> 80.0; bitwise-equal results)
  const int prw_mode = env_int("SMG_PRW", 1);
  t->prw = (prw_mode == 2 || (prw_mode == 1 && p_f == 32)) ? prw_dispatch(p_c, p_f) : nullptr;
  t->J.assign(J, J + (p_f + 1) * (p_c + 1));
  *h = t;
  return SMG_OK;
}

int smg_transfer_destroy(smg_transfer_t* h) { delete h; return SMG_OK; }

static int tr_run(const smg_transfer_t* h, const double* src, double* dst, int acc, bool prolong, cudaStream_t st) {
  TrArgs A;
  std::memset(&A, 0, sizeof(A));
  A.src = src; A.dst = dst; A.n_x = h->n_x; A.n_y = h->n_y; A.accumulate = acc;
  std::memcpy(A.J, h->J.data(), sizeof(double) * h->J.size());
  if (prolong && h->prw) return h->prw(A, st);
  return h->fn(A, h->n_x, h->n_y, prolong, st);
}

int smg_prolongate(const smg_transfer_t* h, const double* uc, double* uf, int accumulate, void* stream) {
  if (!h || !uc || !uf) { set_error("smg_prolongate: bad argument"); return SMG_EINVAL; }
  return tr_run(h, uc, uf, accumulate, true, as_stream(stream));
}

int smg_prolongate_chain(const smg_transfer_t* const* tr, int K, const double* u0, double* const* u,
                         void* stream) {
  if (!tr || !u0 || !u || K < 1) { set_error("smg_prolongate_chain: bad argument"); return SMG_EINVAL; }
  if (K > 4) { set_error("smg_prolongate_chain: chains up to p = 16"); return SMG_EUNSUPPORTED; }
  const double* J[5] = {nullptr};
  double* uu[5] = {nullptr};
  for (int l = 1; l <= K; ++l) {
    const smg_transfer_t* t = tr[l - 1];
    if (!t || !u[l - 1] || t->pc != (1 << (l - 1)) || t->pf != (1 << l) || t->n_x != tr[0]->n_x ||
        t->n_y != tr[0]->n_y) {
      set_error("smg_prolongate_chain: level %d is not the p = %d -> %d transfer of one mesh", l, 1 << (l - 1),
                1 << l);
      return SMG_EUNSUPPORTED;
    }
    J[l] = t->J.data();
    uu[l] = u[l - 1];
  }
  return prolong_chain_run(K, tr[0]->n_x, tr[0]->n_y, J, u0, uu, as_stream(stream));
}

int smg_restrict(const smg_transfer_t* h, const double* ff, double* fc, void* stream) {
  if (!h || !ff || !fc) { set_error("smg_restrict: bad argument"); return SMG_EINVAL; }
  return tr_run(h, ff, fc, 0, false, as_stream(stream));
}

size_t smg_transfer_ws_doubles(const smg_transfer_t* h) {
  return (h && (h->rw || h->rr_opw)) ? (size_t)h->n_x * h->n_y * (2 * h->pc + 1) : 0;
}

int smg_restrict_ws(const smg_transfer_t* h, const double* ff, double* fc, double* ws, void* stream) {
  if (!h || !ff || !fc) { set_error("smg_restrict_ws: bad argument"); return SMG_EINVAL; }
  if (!h->rw || !ws) return smg_restrict(h, ff, fc, stream);
  TrArgs A;
  std::memset(&A, 0, sizeof(A));
  A.src = ff; A.dst = fc; A.n_x = h->n_x; A.n_y = h->n_y;
  std::memcpy(A.J, h->J.data(), sizeof(double) * h->J.size());
  return h->rw(A, ws, as_stream(stream));
}

int smg_residual_restrict_ws(const smg_transfer_t* h, const smg_op_t* op, const double* u, const double* f,
                             double* fc, double* work, double* ws, double* op_ring, void* stream) {
  const bool ring = op && op_ring && smg_op_ring_doubles(op) > 0;
  // Poisson p_f = 16: the warp-per-element residual kernel restricts its element in place
  // (r is neither written nor re-read) and hands the high-side coarse nodes to the ring
  if (h && h->rr_opw && ws && op && u && f && fc && op->kind == 0 && op->p == h->pf && 2 * h->pc == h->pf &&
      op->n_x == h->n_x && op->n_y == h->n_y && h->n_x % 2 == 0 && h->n_y % 2 == 0) {
    OpLaunch L;
    L.u = u; L.f = f; L.out = work; L.nu = op->nu; L.partials = nullptr;
    L.p = op->p; L.n_x = op->n_x; L.n_y = op->n_y; L.diffusion = op->kind;
    L.cx = op->dy / op->dx; L.cy = op->dx / op->dy;
    L.Mt = op->Mt.data(); L.w = op->w.data(); L.wasm = op->wasm.data();
    const int rc = opw_residual_restrict(L, h->J.data(), fc, ws, as_stream(stream));
    if (rc == 0) return rw_fixup(h->pc, fc, ws, h->n_x, h->n_y, as_stream(stream));
    if (rc != 1) return rc;
  }
  if (!h || ((!h->rw || !ws) && !ring)) return smg_residual_restrict(h, op, u, f, fc, work, stream);
  if (!op || !u || !f || !fc || !work) { set_error("smg_residual_restrict_ws: bad argument"); return SMG_EINVAL; }
  int rc = smg_op_residual_ws(op, u, f, work, op_ring, stream);
  if (rc) return rc;
  return smg_restrict_ws(h, work, fc, ws, stream);
}

int smg_residual_restrict(const smg_transfer_t* h, const smg_op_t* op, const double* u, const double* f,
                          double* fc, double* work, void* stream) {
  if (!h || !op || !u || !f || !fc || !work) { set_error("smg_residual_restrict: bad argument"); return SMG_EINVAL; }
  // fused single launch (r never leaves shared memory) when compiled in and
  // the fields allow 16-byte bulk row copies
  // measured (tools/vcycle_breakdown.py, C2): fused wins at p_f <= 8 (4.3 vs
  // 6.9 us at p_f = 2), loses at p_f = 16 (33 vs 22 us: 2.25x residual
  // recompute, 63 KB tiles); SMG_RR_FUSED = 0 never, 1 p_f <= 8, 2 always,
  // 3 p_f <= 4
  static const int fused = env_int("SMG_RR_FUSED", 1);
  if ((fused == 2 || (fused == 1 && h->pf <= 8) || (fused == 3 && h->pf <= 4)) && op->p == h->pf && op->n_x == h->n_x && op->n_y == h->n_y && ((long)h->n_x * h->pf) % 2 == 0) {
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    RRFn fn = rr_dispatch(h->pc, h->pf, op->kind != 0, h->n_x, h->n_y);
    if (fn && al16(u) && al16(f) && (op->kind == 0 || al16(op->nu))) {
      RRLaunch R;
      R.op.u = u; R.op.f = f; R.op.out = nullptr; R.op.nu = op->nu; R.op.partials = nullptr;
      R.op.p = op->p; R.op.n_x = op->n_x; R.op.n_y = op->n_y; R.op.diffusion = op->kind;
      R.op.cx = op->dy / op->dx; R.op.cy = op->dx / op->dy;
      R.op.Mt = op->Mt.data(); R.op.w = op->w.data(); R.op.wasm = op->wasm.data();
      R.fc = fc;
      R.J = h->J.data();
      return fn(R, as_stream(stream));
    }
  }
  int rc = smg_op_residual(op, u, f, work, stream);
  if (rc) return rc;
  return smg_restrict(h, work, fc, stream);
}

// ---- coarse pseudo-inverse -----------------------------------------------------
static void fourier_basis(int n, std::vector<double>& Q, std::vector<double>& mu) {
  // Orthonormal real eigenbasis of the periodic tridiag(-1, 2, -1); column-major
  // by mode: Q[j*n + k] = q_k(j).
  Q.assign((size_t)n * n, 0.0);
  mu.assign(n, 0.0);
  const double pi = 3.14159265358979323846;
  int col = 0;
  for (int j = 0; j < n; ++j) Q[(size_t)j * n + col] = 1.0 / std::sqrt((double)n);
  mu[col++] = 0.0;
  for (int k = 1; 2 * k < n; ++k) {
    const double lam = 2.0 - 2.0 * std::cos(2.0 * pi * k / n);
    for (int j = 0; j < n; ++j) {
      Q[(size_t)j * n + col] = std::sqrt(2.0 / n) * std::cos(2.0 * pi * (double)j * k / n);
      Q[(size_t)j * n + col + 1] = std::sqrt(2.0 / n) * std::sin(2.0 * pi * (double)j * k / n);
    }
    mu[col] = mu[col + 1] = lam;
    col += 2;
  }
  if (n % 2 == 0) {
    for (int j = 0; j < n; ++j) Q[(size_t)j * n + col] = (j % 2 ? -1.0 : 1.0) / std::sqrt((double)n);
    mu[col++] = 4.0;
  }
}

int smg_coarse_create(smg_coarse_t** h, int n_x, int n_y, double dx, double dy) {
  if (!h || n_x < 2 || n_y < 2 || !(dx > 0) || !(dy > 0)) { set_error("smg_coarse_create: bad argument"); return SMG_EINVAL; }
  std::vector<double> Qx, Qy, mx, my;
  fourier_basis(n_x, Qx, mx);
  fourier_basis(n_y, Qy, my);
  std::vector<double> Lp((size_t)n_y * n_x);
  for (int ky = 0; ky < n_y; ++ky)
    for (int kx = 0; kx < n_x; ++kx) {
      const double lam = (dy / dx) * mx[kx] + (dx / dy) * my[ky];
      Lp[(size_t)ky * n_x + kx] = (ky == 0 && kx == 0) ? 0.0 : 1.0 / lam;
    }
  smg_coarse* c = new (std::nothrow) smg_coarse();
  if (!c) return SMG_ENOMEM;
  c->n_x = n_x; c->n_y = n_y; c->dx = dx; c->dy = dy;
  std::vector<double> QxT(Qx.size());
  for (int i = 0; i < n_x; ++i)
    for (int j = 0; j < n_x; ++j) QxT[(size_t)j * n_x + i] = Qx[(size_t)i * n_x + j];
  c->QxT = nullptr;
  cudaError_t e = cudaMalloc(&c->Qx, sizeof(double) * Qx.size());
  if (e == cudaSuccess) e = cudaMalloc(&c->QxT, sizeof(double) * QxT.size());
  if (e == cudaSuccess) e = cudaMemcpy(c->QxT, QxT.data(), sizeof(double) * QxT.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&c->Qy, sizeof(double) * Qy.size());
  if (e == cudaSuccess) e = cudaMalloc(&c->Lp, sizeof(double) * Lp.size());
  if (e == cudaSuccess) e = cudaMemcpy(c->Qx, Qx.data(), sizeof(double) * Qx.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(c->Qy, Qy.data(), sizeof(double) * Qy.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(c->Lp, Lp.data(), sizeof(double) * Lp.size(), cudaMemcpyHostToDevice);
  const std::vector<double> ft = fft_table(n_x, n_y);
  if (e == cudaSuccess && !ft.empty()) {
    e = cudaMalloc(&c->fft, sizeof(double) * ft.size());
    if (e == cudaSuccess) e = cudaMemcpy(c->fft, ft.data(), sizeof(double) * ft.size(), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) { delete c; return cuda_fail(e, "smg_coarse_create"); }
  *h = c;
  return SMG_OK;
}

int smg_coarse_destroy(smg_coarse_t* h) {
  if (!h) return SMG_OK;
  cudaFree(h->Qx); cudaFree(h->QxT); cudaFree(h->Qy); cudaFree(h->Lp);
  if (h->fft) cudaFree(h->fft);
  delete h;
  return SMG_OK;
}

size_t smg_coarse_ws_doubles(const smg_coarse_t* h) { return h ? 2 * (size_t)h->n_x * h->n_y : 0; }

int smg_coarse_pinv(const smg_coarse_t* h, const double* f0, double* u0, double* ws, void* stream) {
  if (!h || !f0 || !u0 || !ws || f0 == u0) { set_error("smg_coarse_pinv: bad argument"); return SMG_EINVAL; }
  cudaStream_t st = as_stream(stream);
  const int nx = h->n_x, ny = h->n_y;
  double* T1 = ws;
  double* T2 = ws + (size_t)nx * ny;
  // power-of-two meshes: 2D FFT (one launch up to 64 x 64, three beyond)
  int rf = pinv_fft(nx, ny, h->dx, h->dy, f0, u0, ws, h->fft, st);
  if (rf != 1) return rf;
  // single-launch cluster variant (SMG_PINV_CLUSTER=0 selects the two-launch
  // row-block path)
  int rc = !(getenv("SMG_PINV_CLUSTER") && getenv("SMG_PINV_CLUSTER")[0] == '0')
               ? pinv_cluster(nx, ny, h->Qx, h->QxT, h->Qy, h->Lp, f0, u0, st) : 1;
  if (rc != 1) return rc;
  rc = pinv_small(nx, ny, h->Qx, h->Qy, h->Lp, f0, T1, u0, st);
  if (rc != 1) return rc;
  // T1 = Qy^T F ; T2 = (T1 Qx) .* Lp ; T1 = Qy T2 ; U = T1 Qx^T
  if ((rc = gemm(ny, nx, ny, h->Qy, ny, 1, f0, nx, 0, T1, nx, nullptr, st))) return rc;
  if ((rc = gemm(ny, nx, nx, T1, nx, 0, h->Qx, nx, 0, T2, nx, h->Lp, st))) return rc;
  if ((rc = gemm(ny, nx, ny, h->Qy, ny, 0, T2, nx, 0, T1, nx, nullptr, st))) return rc;
  return gemm(ny, nx, nx, T1, nx, 0, h->Qx, nx, 1, u0, nx, nullptr, st);
}


// ---- coarse plain CG (parity mode): multigrid.py:196-228 on the device ------
size_t smg_coarse_cg_ws_doubles(int64_t n) { return 4 * (size_t)n + smg_reduce_ws_doubles() + 16; }

int smg_coarse_cg(const smg_op_t* op, const double* f0, double* u0, double* ws, double tol, int max_iter,
                  int* iters_out, void* stream) {
  if (!op || !f0 || !u0 || !ws || !iters_out || op->p != 1 || max_iter < 1) {
    set_error("smg_coarse_cg: bad argument");
    return SMG_EINVAL;
  }
  cudaStream_t st = as_stream(stream);
  const int64_t n = (int64_t)op->n_x * op->n_y;
  double* b = ws;
  double* r = b + n;
  double* p = r + n;
  double* q = p + n;
  double* red = q + n;
  double* S = red + smg_reduce_ws_doubles();
  int rc;
  cudaError_t e;
  // Poisson meshes up to 64 x 64: the whole CG in one CTA (smg_blas.cu
  // ccg_cta_kernel), one host read for the iteration count
  static const int cta = env_int("SMG_CCG_CTA", 1);
  if (cta && op->kind == 0 && n <= 4096) {
    rc = ccg_cta_run(op->n_x, op->n_y, op->dy / op->dx, op->dx / op->dy, f0, u0, tol, max_iter, S, st);
    if (rc != SMG_EUNSUPPORTED) {
      if (rc) return rc;
      double hs[6];
      if ((e = cudaMemcpyAsync(hs, S, sizeof(double) * 6, cudaMemcpyDeviceToHost, st))) return cuda_fail(e, "smg_coarse_cg");
      if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "smg_coarse_cg");
      *iters_out = hs[4] != 0.0 ? (int)hs[5] : -max_iter;
      return SMG_OK;
    }
  }
  // b = f0 - mean(f0); x = 0; r = b; p = r
  if ((e = cudaMemcpyAsync(b, f0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st))) return cuda_fail(e, "smg_coarse_cg");
  if ((rc = smg_project_mean(b, n, red, stream))) return rc;
  if ((e = cudaMemsetAsync(S, 0, sizeof(double) * 16, st))) return cuda_fail(e, "smg_coarse_cg");
  if ((e = cudaMemsetAsync(u0, 0, sizeof(double) * n, st))) return cuda_fail(e, "smg_coarse_cg");
  if ((e = cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st))) return cuda_fail(e, "smg_coarse_cg");
  if ((e = cudaMemcpyAsync(p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st))) return cuda_fail(e, "smg_coarse_cg");
  if ((rc = ccg_dot(b, b, n, S + 0, nullptr, red, st))) return rc;
  if ((rc = ccg_dot(r, r, n, S + 2, nullptr, red, st))) return rc;
  double hs[6];
  if ((e = cudaMemcpyAsync(hs, S, sizeof(double) * 6, cudaMemcpyDeviceToHost, st))) return cuda_fail(e, "smg_coarse_cg");
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "smg_coarse_cg");
  if (hs[0] == 0.0) { *iters_out = 0; return SMG_OK; }
  int it = 0;
  const int chunk = 32;
  while (it < max_iter) {
    const int stop = it + chunk < max_iter ? it + chunk : max_iter;
    for (; it < stop; ++it) {
      const int ro = 2 + (it & 1), rn = 3 - (it & 1);
      if ((rc = smg_op_residual(op, p, nullptr, q, stream))) return rc;
      if ((rc = ccg_dot(p, q, n, S + 1, S, red, st))) return rc;
      if ((rc = ccg_update(u0, r, p, q, n, S, ro, rn, tol, it + 1, red, st))) return rc;
      if ((rc = ccg_direction(p, r, n, S, ro, rn, st))) return rc;
    }
    if ((e = cudaMemcpyAsync(hs, S, sizeof(double) * 6, cudaMemcpyDeviceToHost, st))) return cuda_fail(e, "smg_coarse_cg");
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "smg_coarse_cg");
    if (hs[4] != 0.0) break;
  }
  const bool ok = hs[4] != 0.0;
  *iters_out = ok ? (int)hs[5] : -max_iter;
  // u0 = x - mean(x)  (multigrid.py:228)
  return smg_project_mean(u0, n, red, stream);
}


// ---- coarse PCG (fast mode for variable diffusion) -----------------------------
size_t smg_coarse_pcg_ws_doubles(const smg_coarse_t* h) {
  return h ? 5 * (size_t)h->n_x * h->n_y + smg_coarse_ws_doubles(h) + smg_reduce_ws_doubles() + 16 : 0;
}

int smg_coarse_pcg(const smg_op_t* op, const smg_coarse_t* pc, const double* f0, double* u0, double* ws,
                   double tol, int max_iter, double scale, int* iters_out, void* stream) {
  if (!op || !pc || !f0 || !u0 || !ws || !iters_out || op->p != 1 || op->n_x != pc->n_x || op->n_y != pc->n_y ||
      max_iter < 1) {
    set_error("smg_coarse_pcg: bad argument");
    return SMG_EINVAL;
  }
  cudaStream_t st = as_stream(stream);
  const int64_t n = (int64_t)op->n_x * op->n_y;
  double* b = ws;
  double* r = b + n;
  double* p = r + n;
  double* q = p + n;
  double* z = q + n;
  double* pws = z + n;
  double* red = pws + smg_coarse_ws_doubles(pc);
  double* S = red + smg_reduce_ws_doubles();
  int rc;
  cudaError_t e;
  // preconditioner: the diagonally scaled pseudo-inverse D^-1/2 A_P^+ D^-1/2
  // (D = nodal nu; SPD on the range of A_0 -- its null space sqrt(nu) is not
  // in it): at C5 11 iterations instead of 59 for the 1/mean(nu)-scaled A_P^+
  // (SMG_PCG_DIAG=0), coarse solve 4.95 -> 1.32 ms on B200; q is free while
  // the preconditioner runs
  static const int diag = env_int("SMG_PCG_DIAG", 1);
  const bool dsc = diag && op->kind == 1 && op->nu != nullptr;
  auto precond = [&](const double* in, double* out) -> int {
    if (dsc) {
      int rr = pcg_dscale(in, q, op->nu, n, S, st);
      if (!rr) rr = smg_coarse_pinv(pc, q, out, pws, stream);
      if (!rr) rr = pcg_dscale(out, out, op->nu, n, S, st);
      return rr;
    }
    int rr = smg_coarse_pinv(pc, in, out, pws, stream);
    if (rr) return rr;
    return pcg_scale(out, n, scale, S, st);
  };
  if ((e = cudaMemcpyAsync(b, f0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st))) return cuda_fail(e, "smg_coarse_pcg");
  if ((rc = smg_project_mean(b, n, red, stream))) return rc;
  if ((e = cudaMemsetAsync(S, 0, sizeof(double) * 16, st))) return cuda_fail(e, "smg_coarse_pcg");
  if ((e = cudaMemsetAsync(u0, 0, sizeof(double) * n, st))) return cuda_fail(e, "smg_coarse_pcg");
  if ((e = cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st))) return cuda_fail(e, "smg_coarse_pcg");
  if ((rc = ccg_dot(b, b, n, S + 0, nullptr, red, st))) return rc;
  if ((rc = precond(r, z))) return rc;
  if ((e = cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, st))) return cuda_fail(e, "smg_coarse_pcg");
  if ((rc = ccg_dot(r, z, n, S + 2, nullptr, red, st))) return rc;
  double hs[8];
  if ((e = cudaMemcpyAsync(hs, S, sizeof(double) * 8, cudaMemcpyDeviceToHost, st))) return cuda_fail(e, "smg_coarse_pcg");
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "smg_coarse_pcg");
  if (hs[0] == 0.0) { *iters_out = 0; return SMG_OK; }
  int it = 0;
  // the whole iteration loop as one cooperative kernel (smg_fft.cu pcg_coop_kernel) where it
  // applies: diagonally scaled FFT preconditioner, power-of-two mesh of 128..512 nodes a side.
  // b and q are free by now: the per-CTA partial sums and the second p buffer
  if (dsc) {
    rc = pcg_coop(pc->n_x, pc->n_y, pc->dx, pc->dy, pc->fft, op->nu, u0, r, p, q, z, pws, b, S, tol, max_iter, st);
    if (rc != 1) {
      if (rc) return rc;
      if ((e = cudaMemcpyAsync(hs, S, sizeof(double) * 8, cudaMemcpyDeviceToHost, st))) return cuda_fail(e, "smg_coarse_pcg");
      if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "smg_coarse_pcg");
      const bool okc = hs[4] != 0.0;
      *iters_out = okc ? (int)hs[5] : -max_iter;
      return smg_project_mean(u0, n, red, stream);
    }
  }
  // iterations between two host reads of the convergence flag: the iterations enqueued
  // after convergence still run (C5: 11-14 needed; with one read per 16 iterations 2-5 of
  // 16 were wasted, ~80 us each), so after the first 8 the flag is read every 3
  static const int chunk0 = env_int("SMG_PCG_CHUNK0", 8), chunk1 = env_int("SMG_PCG_CHUNK", 3);
  while (it < max_iter) {
    const int chunk = it == 0 ? chunk0 : chunk1;
    const int stop = it + chunk < max_iter ? it + chunk : max_iter;
    for (; it < stop; ++it) {
      const int ro = 2 + (it & 1), rn = 3 - (it & 1);
      if ((rc = smg_op_residual(op, p, nullptr, q, stream))) return rc;
      if ((rc = ccg_dot(p, q, n, S + 1, S, red, st))) return rc;
      if ((rc = pcg_update(u0, r, p, q, n, S, ro, tol, it + 1, red, st))) return rc;
      if ((rc = precond(r, z))) return rc;
      if ((rc = ccg_dot(r, z, n, S + rn, S, red, st))) return rc;
      if ((rc = ccg_direction(p, z, n, S, ro, rn, st))) return rc;
    }
    if ((e = cudaMemcpyAsync(hs, S, sizeof(double) * 8, cudaMemcpyDeviceToHost, st))) return cuda_fail(e, "smg_coarse_pcg");
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "smg_coarse_pcg");
    if (hs[4] != 0.0) break;
  }
  const bool ok = hs[4] != 0.0;
  *iters_out = ok ? (int)hs[5] : -max_iter;
  return smg_project_mean(u0, n, red, stream);
}


}  // extern "C"

// ---- multiplicative Schwarz (smg_mult.cu) -----------------------------------

struct smg_mult {
  int p, n_o, n_x, n_y, m;
  const double* nu_bar;   // caller's device (n_y, n_x), nullable
  std::vector<void*> owned;
  const double *Sx, *Sy, *dinv;
};

extern "C" {

int smg_mult_destroy(smg_mult_t* h) {
  if (!h) return SMG_OK;
  for (void* p : h->owned) cudaFree(p);
  delete h;
  return SMG_OK;
}

int smg_mult_create(smg_mult_t** out, int p, int n_o, int n_x, int n_y, const double* S_x, const double* S_y,
                    const double* lam_x, const double* lam_y, const double* nu_bar_dev) {
  if (!out || !S_x || !S_y || !lam_x || !lam_y || p < 1 || n_o < 0 || n_o > p - 1 || n_x < 1 || n_y < 1) {
    set_error("smg_mult_create: bad argument");
    return SMG_EINVAL;
  }
  const int m = p + 1 + 2 * n_o;
  if (m > p * n_x || m > p * n_y) {
    set_error("subdomain window (%d nodes) wraps onto itself on a %dx%d mesh at p=%d; reduce n_o", m, n_x, n_y, p);
    return SMG_EINVAL;
  }
  smg_mult* h = new (std::nothrow) smg_mult();
  if (!h) return SMG_ENOMEM;
  h->p = p; h->n_o = n_o; h->n_x = n_x; h->n_y = n_y; h->m = m; h->nu_bar = nu_bar_dev;
  std::vector<double> dinv((size_t)m * m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) dinv[(size_t)i * m + j] = 1.0 / (lam_y[i] + lam_x[j]);
  auto upload = [&](const double* src, size_t n, const double** dst) -> cudaError_t {
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(double) * n);
    if (e != cudaSuccess) return e;
    h->owned.push_back(d);
    *dst = static_cast<const double*>(d);
    return cudaMemcpy(d, src, sizeof(double) * n, cudaMemcpyHostToDevice);
  };
  cudaError_t e = upload(S_x, (size_t)m * m, &h->Sx);
  if (e == cudaSuccess) e = upload(S_y, (size_t)m * m, &h->Sy);
  if (e == cudaSuccess) e = upload(dinv.data(), dinv.size(), &h->dinv);
  if (e != cudaSuccess) { smg_mult_destroy(h); return cuda_fail(e, "smg_mult_create"); }
  *out = h;
  return SMG_OK;
}

int smg_mult_sweep(const smg_mult_t* h, const smg_op_t* op, double* u, double* r, int forward, void* stream) {
  if (!h || !op || !u || !r || u == r || op->p != h->p || op->n_x != h->n_x || op->n_y != h->n_y) {
    set_error("smg_mult_sweep: bad argument");
    return SMG_EINVAL;
  }
  // operator constants in the reference's element_kernel form
  // (operators.py:44-47 Poisson, :80-84 diffusion), by value per launch
  const int NP = h->p + 1;
  if (NP > kMsMaxNP) { set_error("smg_mult_sweep: p=%d beyond %d", h->p, kMsMaxNP - 1); return SMG_EUNSUPPORTED; }
  MsArgs A;
  std::memset(&A, 0, sizeof(A));
  A.u = u; A.r = r; A.Sx = h->Sx; A.Sy = h->Sy; A.dinv = h->dinv; A.nu_bar = h->nu_bar;
  for (int i = 0; i < NP * NP; ++i) {
    A.Ly[i] = op->kind == 0 ? (2.0 / op->dy) * op->Mt[i] : op->Mt[i];
    A.Lx[i] = (2.0 / op->dx) * op->Mt[i];
  }
  for (int i = 0; i < NP; ++i) {
    A.my[i] = (op->dy / 2.0) * op->w[i];
    A.mx[i] = (op->dx / 2.0) * op->w[i];
    A.w[i] = op->w[i];
  }
  A.diffusion = op->kind == 1;
  A.nu = op->kind == 1 ? op->nu : nullptr;
  A.cx = op->dy / op->dx; A.cy = op->dx / op->dy;
  A.p = h->p; A.n_o = h->n_o; A.m = h->m; A.n_x = h->n_x; A.n_y = h->n_y; A.forward = forward ? 1 : 0;
  return mult_sweep_launch(A, as_stream(stream));
}

}  // extern "C"
