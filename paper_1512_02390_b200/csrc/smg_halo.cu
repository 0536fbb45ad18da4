// Strip halos and strip collectives over NCCL: the C ABI
// the multi-GPU V-cycle and MGCG call between the per-level kernels.
//
// The reference is single-process; at a strip boundary these replace the
// periodic wrap of its subdomain windows (mesh.py:124-139
// all_element_windows) and of its operator's element gather (mesh.py:97-105),
// and the global sums of its inner products (krylov.py:91-111, numpy.vdot).
// Rank g owns element rows [g s, (g + 1) s); the rank below is g - 1 and the
// rank above g + 1 (mod nranks), so a one-rank communicator wraps onto
// itself -- the same exchanges then run as NCCL self send/recv.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2": in a PyTorch process
// the copy torch already mapped), so libsmg loads and every single-GPU entry
// point works on a machine without NCCL; the halo calls then fail with
// SMG_EUNSUPPORTED.  Every call enqueues on the caller's stream and never
// synchronizes, so a strip V-cycle including its halos can be captured into
// one CUDA graph.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "smg_common.cuh"

struct smg_halo {
  ncclComm_t comm;
  int nranks, rank, device;
};

namespace smg {
namespace {

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
  bool ok = false;
};

const Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SMG_NCCL_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
    SMG_NCCL_SYM(get_unique_id, "ncclGetUniqueId");
    SMG_NCCL_SYM(init_rank, "ncclCommInitRank");
    SMG_NCCL_SYM(destroy, "ncclCommDestroy");
    SMG_NCCL_SYM(group_start, "ncclGroupStart");
    SMG_NCCL_SYM(group_end, "ncclGroupEnd");
    SMG_NCCL_SYM(send, "ncclSend");
    SMG_NCCL_SYM(recv, "ncclRecv");
    SMG_NCCL_SYM(all_reduce, "ncclAllReduce");
    SMG_NCCL_SYM(all_gather, "ncclAllGather");
    SMG_NCCL_SYM(error_string, "ncclGetErrorString");
    SMG_NCCL_SYM(get_version, "ncclGetVersion");
#undef SMG_NCCL_SYM
    n.ok = n.get_unique_id && n.init_rank && n.destroy && n.group_start && n.group_end && n.send && n.recv &&
           n.all_reduce && n.all_gather && n.error_string && n.get_version;
  });
  return n.ok ? &n : nullptr;
}

int need_nccl(const Nccl*& n) {
  n = nccl();
  if (!n) {
    set_error("NCCL is not available (dlopen libnccl.so.2 failed or symbols missing)");
    return SMG_EUNSUPPORTED;
  }
  return SMG_OK;
}

int nccl_fail(const Nccl* n, ncclResult_t r, const char* where) {
  set_error("%s: NCCL error %d (%s)", where, (int)r, n->error_string(r));
  return SMG_ECUDA;
}

#define SMG_NCCL_TRY(call, where)                 \
  do {                                            \
    ncclResult_t r_ = (call);                     \
    if (r_ != ncclSuccess) return nccl_fail(n, r_, where); \
  } while (0)

int check_halo(const smg_halo* h, const void* t, int64_t rows, int64_t row_len, int64_t lo, int64_t hi, int below,
               int above, const char* where) {
  if (!h || !t || row_len <= 0 || below < 0 || above < 0 || lo < below || hi <= lo || hi + above > rows ||
      above > hi - lo || below > hi - lo) {
    set_error("%s: bad arguments (%lld rows of %lld, owned rows [%lld, %lld), below %d, above %d)", where,
              (long long)rows, (long long)row_len, (long long)lo, (long long)hi, below, above);
    return SMG_EINVAL;
  }
  return SMG_OK;
}

// one exchange: send_down -> rank below, recv_from_above <- rank above (n_a
// doubles each), send_up -> rank above, recv_from_below <- rank below (n_b).
// Sends and receives are issued in this fixed order on every rank, so with
// two ranks (below == above) the k-th send to a peer matches the peer's k-th
// receive from it, and with one rank the self send/recv pairs match.
int p2p(const Nccl* n, const smg_halo* h, const double* send_down, double* recv_from_above, size_t n_a,
        const double* send_up, double* recv_from_below, size_t n_b, cudaStream_t st, const char* where) {
  if (n_a == 0 && n_b == 0) return SMG_OK;
  const int below = (h->rank + h->nranks - 1) % h->nranks, above = (h->rank + 1) % h->nranks;
  SMG_NCCL_TRY(n->group_start(), where);
  if (n_a) {
    SMG_NCCL_TRY(n->send(send_down, n_a, ncclDouble, below, h->comm, st), where);
    SMG_NCCL_TRY(n->recv(recv_from_above, n_a, ncclDouble, above, h->comm, st), where);
  }
  if (n_b) {
    SMG_NCCL_TRY(n->send(send_up, n_b, ncclDouble, above, h->comm, st), where);
    SMG_NCCL_TRY(n->recv(recv_from_below, n_b, ncclDouble, below, h->comm, st), where);
  }
  SMG_NCCL_TRY(n->group_end(), where);
  return SMG_OK;
}

// t[r][c] for owned rows r in [lo, hi): + from_below on [lo, lo + above),
// then + from_above on [hi - below, hi) -- one pass, the two additions in this
// fixed order on a row both ranges cover (a thin strip).
__global__ void halo_add_kernel(double* __restrict__ t, int64_t row_len, int64_t lo, int64_t hi, int below,
                                int above, const double* __restrict__ from_below,
                                const double* __restrict__ from_above) {
  SMG_PDL_ENTRY();
  const bool joined = lo + above >= hi - below;          // the two ranges meet: one span [lo, hi)
  const int64_t rows = joined ? hi - lo : (int64_t)above + below;
  const int64_t total = rows * row_len;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = k / row_len, c = k - j * row_len;
    const int64_t row = (joined || j < above) ? lo + j : hi - below + (j - above);
    double v = t[row * row_len + c];
    if (row < lo + above) v += from_below[(row - lo) * row_len + c];
    if (row >= hi - below) v += from_above[(row - (hi - below)) * row_len + c];
    t[row * row_len + c] = v;
  }
}

}  // namespace
}  // namespace smg

using namespace smg;

extern "C" {

int smg_halo_available(void) { return nccl() != nullptr; }

int smg_halo_unique_id(unsigned char* out, int n_bytes) {
  const Nccl* n;
  if (int rc = need_nccl(n)) return rc;
  if (!out || n_bytes < (int)sizeof(ncclUniqueId)) {
    set_error("smg_halo_unique_id: need %d bytes", (int)sizeof(ncclUniqueId));
    return SMG_EINVAL;
  }
  ncclUniqueId id;
  SMG_NCCL_TRY(n->get_unique_id(&id), "smg_halo_unique_id");
  std::memcpy(out, &id, sizeof(id));
  return SMG_OK;
}

int smg_halo_create(const unsigned char* id, int n_bytes, int nranks, int rank, int device, smg_halo_t** out) {
  const Nccl* n;
  if (int rc = need_nccl(n)) return rc;
  if (!id || n_bytes < (int)sizeof(ncclUniqueId) || nranks < 1 || rank < 0 || rank >= nranks || !out) {
    set_error("smg_halo_create: bad arguments (nranks %d, rank %d)", nranks, rank);
    return SMG_EINVAL;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "smg_halo_create");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  SMG_NCCL_TRY(n->init_rank(&comm, nranks, uid, rank), "smg_halo_create");
  *out = new smg_halo{comm, nranks, rank, device};
  return SMG_OK;
}

int smg_halo_destroy(smg_halo_t* h) {
  if (!h) return SMG_OK;
  const Nccl* n;
  if (int rc = need_nccl(n)) return rc;
  ncclResult_t r = n->destroy(h->comm);
  delete h;
  if (r != ncclSuccess) return nccl_fail(n, r, "smg_halo_destroy");
  return SMG_OK;
}

int smg_halo_nccl_version(void) {
  const Nccl* n = nccl();
  int v = 0;
  if (!n || n->get_version(&v) != ncclSuccess) return 0;
  return v;
}

int64_t smg_halo_ws_doubles(int64_t row_len, int below, int above) {
  return row_len * (int64_t)(below + above);
}

int smg_halo_exchange(const smg_halo_t* h, double* t, int64_t rows, int64_t row_len, int64_t lo, int64_t hi,
                      int below, int above, void* stream) {
  const Nccl* n;
  if (int rc = need_nccl(n)) return rc;
  if (int rc = check_halo(h, t, rows, row_len, lo, hi, below, above, "smg_halo_exchange")) return rc;
  // my bottom `above` owned rows are the lower neighbour's top ghost rows, my
  // top `below` owned rows the upper neighbour's bottom ghost rows
  return p2p(n, h, t + lo * row_len, t + hi * row_len, (size_t)above * row_len, t + (hi - below) * row_len,
             t + (lo - below) * row_len, (size_t)below * row_len, as_stream(stream), "smg_halo_exchange");
}

int smg_halo_exchange_add(const smg_halo_t* h, double* t, int64_t rows, int64_t row_len, int64_t lo, int64_t hi,
                          int below, int above, double* ws, void* stream) {
  const Nccl* n;
  if (int rc = need_nccl(n)) return rc;
  if (int rc = check_halo(h, t, rows, row_len, lo, hi, below, above, "smg_halo_exchange_add")) return rc;
  if (!ws) {
    set_error("smg_halo_exchange_add: workspace of smg_halo_ws_doubles() doubles required");
    return SMG_EINVAL;
  }
  if (below == 0 && above == 0) return SMG_OK;
  // the ghost rows under the strip belong to the rank below (its top owned
  // rows), the ghost rows over it to the rank above
  double* from_above = ws;                          // `below` rows: the upper rank's bottom ghosts
  double* from_below = ws + (int64_t)below * row_len;  // `above` rows: the lower rank's top ghosts
  cudaStream_t st = as_stream(stream);
  if (int rc = p2p(n, h, t + (lo - below) * row_len, from_above, (size_t)below * row_len, t + hi * row_len,
                   from_below, (size_t)above * row_len, st, "smg_halo_exchange_add"))
    return rc;
  const int64_t total = (int64_t)(below + above) * row_len;
  const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  launch(halo_add_kernel, dim3(grid), dim3(256), 0, st, t, row_len, lo, hi, below, above,
         (const double*)from_below, (const double*)from_above);
  return check_launch("halo_add_kernel");
}

int smg_halo_allreduce(const smg_halo_t* h, double* x, int64_t n_el, void* stream) {
  const Nccl* n;
  if (int rc = need_nccl(n)) return rc;
  if (!h || !x || n_el < 0) {
    set_error("smg_halo_allreduce: bad arguments");
    return SMG_EINVAL;
  }
  if (n_el == 0) return SMG_OK;
  SMG_NCCL_TRY(n->all_reduce(x, x, (size_t)n_el, ncclDouble, ncclSum, h->comm, as_stream(stream)),
               "smg_halo_allreduce");
  return SMG_OK;
}

int smg_halo_allgather(const smg_halo_t* h, const double* own, double* full, int64_t n_per_rank, void* stream) {
  const Nccl* n;
  if (int rc = need_nccl(n)) return rc;
  if (!h || !own || !full || n_per_rank < 0) {
    set_error("smg_halo_allgather: bad arguments");
    return SMG_EINVAL;
  }
  if (n_per_rank == 0) return SMG_OK;
  SMG_NCCL_TRY(n->all_gather(own, full, (size_t)n_per_rank, ncclDouble, h->comm, as_stream(stream)),
               "smg_halo_allgather");
  return SMG_OK;
}

}  // extern "C"
