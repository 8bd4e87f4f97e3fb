// Multi-GPU boundary of the C ABI ("ldg_comm_init(ncclComm_t,
// partition), with halo exchange issued inside the matvec calls").
//
// One handle per rank holds the rank's owned elements plus a ghost layer
// (the caller's partition: PartitionPlan in parallel.py); ldg_set_halo_plan
// gives the face-node halo lists (which owned (element, node) rows go to
// which peer, where received rows land in the ghost buffer) and the export
// lists of pass 2 (element-face slots of X).  ldg_apply_dist then runs the
// operator with both exchanges inside the call:
//
//   pack u rows -> [comm stream] send / recv    | pass 1 on the interior range
//   unpack into the ghost rows; pass 1 on the rest
//   pack X rows -> [comm stream] send / recv    | pass 2 on the interior range
//   unpack into X; pass 2 on the rest
//
// Transports: NCCL (ldg_comm_init: ncclCommInitRank from a unique id the
// caller broadcasts; grouped ncclSend / ncclRecv of device buffers on the
// comm stream; libnccl is dlopen'ed -- the process's already loaded NCCL
// first -- so the library itself has no link dependency), or in-process
// (ldg_comm_init_local: several handles on one device, each driven from
// its own host thread like a rank; device-to-device copies into the peer's
// receive buffer, ordered by CUDA events and a host-side mailbox).  Both
// use the same pack / unpack kernels, plan and overlap schedule.

#include <dlfcn.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "ldgb200.h"
#include "nvtx.cuh"

namespace ldg {
int set_error(int code, const char* what, cudaError_t e);
}

namespace {

// ---- NCCL, resolved at run time ---------------------------------------------
typedef struct { char internal[128]; } NcclId;
typedef void* NcclComm;
typedef int (*fn_get_id)(NcclId*);
typedef int (*fn_init_rank)(NcclComm*, int, NcclId, int);
typedef int (*fn_destroy)(NcclComm);
typedef int (*fn_sendrecv)(const void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*fn_recv)(void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*fn_group)(void);
typedef const char* (*fn_errstr)(int);
constexpr int kNcclDouble = 8;                 // ncclFloat64

struct Nccl {
  bool tried = false, ok = false;
  fn_get_id get_id = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_destroy destroy = nullptr;
  fn_sendrecv send = nullptr;
  fn_recv recv = nullptr;
  fn_group group_start = nullptr, group_end = nullptr;
  fn_errstr errstr = nullptr;
};
Nccl g_nccl;
std::mutex g_nccl_m;

bool load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_m);
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);     // torch's, if loaded
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return false;
  g_nccl.get_id = (fn_get_id)dlsym(lib, "ncclGetUniqueId");
  g_nccl.init_rank = (fn_init_rank)dlsym(lib, "ncclCommInitRank");
  g_nccl.destroy = (fn_destroy)dlsym(lib, "ncclCommDestroy");
  g_nccl.send = (fn_sendrecv)dlsym(lib, "ncclSend");
  g_nccl.recv = (fn_recv)dlsym(lib, "ncclRecv");
  g_nccl.group_start = (fn_group)dlsym(lib, "ncclGroupStart");
  g_nccl.group_end = (fn_group)dlsym(lib, "ncclGroupEnd");
  g_nccl.errstr = (fn_errstr)dlsym(lib, "ncclGetErrorString");
  g_nccl.ok = g_nccl.get_id && g_nccl.init_rank && g_nccl.destroy && g_nccl.send &&
              g_nccl.recv && g_nccl.group_start && g_nccl.group_end;
  return g_nccl.ok;
}

int nccl_fail(int r, const char* what) {
  std::string m = std::string(what) + ": " + (g_nccl.errstr ? g_nccl.errstr(r) : "nccl error");
  return ldg::set_error(4, m.c_str(), cudaSuccess);
}

// ---- per-handle state ---------------------------------------------------------
struct Phase {                         // one exchange: u rows (pass 1) or X rows (pass 2)
  int width = 0;                       // doubles per row
  std::vector<int64_t> send_off, recv_off;   // per peer, in rows
  int64_t* send_idx = nullptr;         // device, concatenated over peers
  int64_t* recv_idx = nullptr;
  double* send_buf = nullptr;
  double* recv_buf = nullptr;
  int64_t nsend = 0, nrecv = 0;
};

struct LocalHub;

struct Comm {
  int nranks = 1, rank = 0;
  NcclComm nccl = nullptr;
  LocalHub* hub = nullptr;             // in-process transport
  std::vector<int> peers;              // peer ranks, ascending
  Phase ph[2];
  int ne = 0, ia = 0, ib = 0;          // owned elements, interior range
  double* u_ghost = nullptr;
  cudaStream_t s_comm = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_recv = nullptr;
  bool planned = false;
};

std::mutex g_comm_m;
std::unordered_map<LdgHandle*, Comm*> g_comms;

Comm* comm_of(LdgHandle* h) {
  std::lock_guard<std::mutex> lk(g_comm_m);
  auto it = g_comms.find(h);
  return it == g_comms.end() ? nullptr : it->second;
}

// ---- in-process transport: mailbox of (src, dst, phase) slots -----------------
struct Slot {
  int64_t sent = 0, consumed = 0;      // rounds posted / unpacked by the receiver
  cudaEvent_t ev_sent = nullptr, ev_consumed = nullptr;
};

struct LocalHub {
  std::mutex m;
  std::condition_variable cv;
  std::vector<LdgHandle*> hs;          // rank -> handle
  std::map<std::tuple<int, int, int>, Slot> box;
  Slot& slot(int src, int dst, int phase) { return box[std::make_tuple(src, dst, phase)]; }
};

int make_comm(LdgHandle* h, Comm** out) {
  Comm* c = new Comm();
  if (cudaStreamCreateWithFlags(&c->s_comm, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_recv, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return ldg::set_error(3, "comm stream / events", cudaGetLastError());
  }
  std::lock_guard<std::mutex> lk(g_comm_m);
  g_comms[h] = c;
  *out = c;
  return 0;
}

void free_phase(Phase& p) {
  cudaFree(p.send_idx);
  cudaFree(p.recv_idx);
  cudaFree(p.send_buf);
  cudaFree(p.recv_buf);
  p = Phase();
}

// ---- pack / unpack -------------------------------------------------------------
__global__ void gather_rows(int64_t n, int w, const int64_t* __restrict__ idx,
                            const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * w;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / w, c = t - r * w;
    dst[t] = src[idx[r] * w + c];
  }
}

__global__ void scatter_rows(int64_t n, int w, const int64_t* __restrict__ idx,
                             const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * w;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / w, c = t - r * w;
    dst[idx[r] * w + c] = src[t];
  }
}

unsigned grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (unsigned)(g < 148 * 8 ? (g > 0 ? g : 1) : 148 * 8);
}

// exchange of one phase on the comm stream (after ev_pack); records ev_recv
int exchange(LdgHandle* h, Comm* c, int phase) {
  Phase& p = c->ph[phase];
  const int np = (int)c->peers.size();
  if (c->nccl) {
    int r = g_nccl.group_start();
    if (r) return nccl_fail(r, "ncclGroupStart");
    for (int k = 0; k < np; ++k) {
      const int64_t ns = p.send_off[k + 1] - p.send_off[k], nr = p.recv_off[k + 1] - p.recv_off[k];
      if (ns && (r = g_nccl.send(p.send_buf + p.send_off[k] * p.width, (size_t)(ns * p.width),
                                 kNcclDouble, c->peers[k], c->nccl, c->s_comm)))
        return nccl_fail(r, "ncclSend");
      if (nr && (r = g_nccl.recv(p.recv_buf + p.recv_off[k] * p.width, (size_t)(nr * p.width),
                                 kNcclDouble, c->peers[k], c->nccl, c->s_comm)))
        return nccl_fail(r, "ncclRecv");
    }
    if ((r = g_nccl.group_end())) return nccl_fail(r, "ncclGroupEnd");
  } else if (c->hub) {
    LocalHub* hub = c->hub;
    // sends: wait until the peer unpacked the previous round, copy into its
    // receive buffer, post
    for (int k = 0; k < np; ++k) {
      const int q = c->peers[k];
      const int64_t ns = p.send_off[k + 1] - p.send_off[k];
      Comm* pc = comm_of(hub->hs[q]);
      int kk = -1;
      for (int j = 0; j < (int)pc->peers.size(); ++j)
        if (pc->peers[j] == c->rank) kk = j;
      if (kk < 0) return ldg::set_error(2, "local peer does not list this rank", cudaSuccess);
      Phase& pp = pc->ph[phase];
      if (pp.recv_off[kk + 1] - pp.recv_off[kk] != ns)
        return ldg::set_error(2, "halo plans disagree on a send / receive count", cudaSuccess);
      std::unique_lock<std::mutex> lk(hub->m);
      Slot& s = hub->slot(c->rank, q, phase);
      hub->cv.wait(lk, [&] { return s.consumed >= s.sent; });
      if (s.ev_consumed) cudaStreamWaitEvent(c->s_comm, s.ev_consumed, 0);
      if (ns && cudaMemcpyAsync(pp.recv_buf + pp.recv_off[kk] * p.width,
                                p.send_buf + p.send_off[k] * p.width,
                                (size_t)ns * p.width * sizeof(double),
                                cudaMemcpyDeviceToDevice, c->s_comm) != cudaSuccess)
        return ldg::set_error(3, "local halo copy", cudaGetLastError());
      if (!s.ev_sent) cudaEventCreateWithFlags(&s.ev_sent, cudaEventDisableTiming);
      cudaEventRecord(s.ev_sent, c->s_comm);
      s.sent += 1;
      hub->cv.notify_all();
    }
    // receives: wait for each peer's post of this round
    for (int k = 0; k < np; ++k) {
      const int q = c->peers[k];
      std::unique_lock<std::mutex> lk(hub->m);
      Slot& s = hub->slot(q, c->rank, phase);
      hub->cv.wait(lk, [&] { return s.sent > s.consumed; });
      cudaStreamWaitEvent(c->s_comm, s.ev_sent, 0);
    }
  }
  if (cudaEventRecord(c->ev_recv, c->s_comm) != cudaSuccess)
    return ldg::set_error(3, "comm event", cudaGetLastError());
  return 0;
}

// receiver side: the unpack of this round is enqueued on `s`; tell the peers
void consumed(Comm* c, int phase, cudaStream_t s) {
  if (!c->hub) return;
  LocalHub* hub = c->hub;
  std::lock_guard<std::mutex> lk(hub->m);
  for (int q : c->peers) {
    Slot& sl = hub->slot(q, c->rank, phase);
    if (!sl.ev_consumed) cudaEventCreateWithFlags(&sl.ev_consumed, cudaEventDisableTiming);
    cudaEventRecord(sl.ev_consumed, s);
    sl.consumed = sl.sent;
  }
  hub->cv.notify_all();
}

int run_phase(LdgHandle* h, Comm* c, int phase, const double* src, double* dst,
              cudaStream_t s, int tangent, const double* u, const double* gproj,
              const double* bsrc, double* X, double* R) {
  Phase& p = c->ph[phase];
  const int pass = phase + 1;
  if (p.nsend)
    gather_rows<<<grid_for(p.nsend * p.width), 256, 0, s>>>(p.nsend, p.width, p.send_idx, src,
                                                              p.send_buf);
  if (cudaEventRecord(c->ev_pack, s) != cudaSuccess ||
      cudaStreamWaitEvent(c->s_comm, c->ev_pack, 0) != cudaSuccess)
    return ldg::set_error(3, "pack event", cudaGetLastError());
  int rc = exchange(h, c, phase);
  if (rc) return rc;
  // interior elements while the halo is in flight
  rc = ldg_operator_pass_range(h, pass, tangent, u, gproj, bsrc, X, R, c->ia, c->ib, s);
  if (rc) return rc;
  if (cudaStreamWaitEvent(s, c->ev_recv, 0) != cudaSuccess)
    return ldg::set_error(3, "recv event", cudaGetLastError());
  if (p.nrecv)
    scatter_rows<<<grid_for(p.nrecv * p.width), 256, 0, s>>>(p.nrecv, p.width, p.recv_idx,
                                                               p.recv_buf, dst);
  consumed(c, phase, s);
  rc = ldg_operator_pass_range(h, pass, tangent, u, gproj, bsrc, X, R, 0, c->ia, s);
  if (!rc) rc = ldg_operator_pass_range(h, pass, tangent, u, gproj, bsrc, X, R, c->ib, c->ne, s);
  return rc;
}

template <typename T>
int up(T** dst, const T* src, int64_t n) {
  *dst = nullptr;
  if (n <= 0) return 0;
  if (cudaMalloc(dst, n * sizeof(T)) != cudaSuccess) return 3;
  if (src && cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess) return 3;
  return 0;
}

}  // namespace

extern "C" {

int ldg_comm_unique_id(uint8_t* id128) {
  if (!id128) return ldg::set_error(2, "null id buffer", cudaSuccess);
  if (!load_nccl()) return ldg::set_error(4, "libnccl.so.2 not found", cudaSuccess);
  NcclId id;
  const int r = g_nccl.get_id(&id);
  if (r) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id128, id.internal, 128);
  return 0;
}

int ldg_comm_init(LdgHandle* h, int nranks, int rank, const uint8_t* id128) {
  NvtxRange nvtx_("ldg_comm_init");
  if (!h || !id128 || nranks < 1 || rank < 0 || rank >= nranks)
    return ldg::set_error(2, "bad argument", cudaSuccess);
  if (comm_of(h)) return ldg::set_error(2, "handle already has a communicator", cudaSuccess);
  if (!load_nccl()) return ldg::set_error(4, "libnccl.so.2 not found", cudaSuccess);
  Comm* c = nullptr;
  int rc = make_comm(h, &c);
  if (rc) return rc;
  c->nranks = nranks;
  c->rank = rank;
  NcclId id;
  memcpy(id.internal, id128, 128);
  const int r = g_nccl.init_rank(&c->nccl, nranks, id, rank);
  if (r) {
    c->nccl = nullptr;
    ldg_comm_destroy(h);
    return nccl_fail(r, "ncclCommInitRank");
  }
  return 0;
}

int ldg_comm_init_local(LdgHandle** hs, int n) {
  if (!hs || n < 1) return ldg::set_error(2, "bad argument", cudaSuccess);
  LocalHub* hub = new LocalHub();
  hub->hs.assign(hs, hs + n);
  for (int r = 0; r < n; ++r) {
    if (!hs[r] || comm_of(hs[r])) return ldg::set_error(2, "null or already linked handle", cudaSuccess);
    Comm* c = nullptr;
    const int rc = make_comm(hs[r], &c);
    if (rc) return rc;
    c->nranks = n;
    c->rank = r;
    c->hub = hub;
  }
  return 0;
}

int ldg_set_halo_plan(LdgHandle* h, int ne_owned, int interior0, int interior1, double* u_ghost,
                      int u_width, int x_width, int npeers, const int32_t* peers,
                      const int64_t* u_send_off, const int64_t* u_send_idx,
                      const int64_t* u_recv_off, const int64_t* u_recv_idx,
                      const int64_t* x_send_off, const int64_t* x_send_idx,
                      const int64_t* x_recv_off, const int64_t* x_recv_idx) {
  Comm* c = comm_of(h);
  if (!c) return ldg::set_error(2, "no communicator: ldg_comm_init first", cudaSuccess);
  if (ne_owned < 0 || interior0 < 0 || interior1 < interior0 || interior1 > ne_owned ||
      u_width < 1 || x_width < 1 || npeers < 0 || (npeers && (!peers || !u_send_off ||
      !u_recv_off || !x_send_off || !x_recv_off)))
    return ldg::set_error(2, "bad halo plan", cudaSuccess);
  for (int k = 0; k < npeers; ++k)
    if (peers[k] < 0 || peers[k] >= c->nranks || peers[k] == c->rank || (k && peers[k] <= peers[k - 1]))
      return ldg::set_error(2, "peers must be distinct other ranks, ascending", cudaSuccess);
  free_phase(c->ph[0]);
  free_phase(c->ph[1]);
  c->ne = ne_owned;
  c->ia = interior0;
  c->ib = interior1;
  c->u_ghost = u_ghost;
  c->peers.assign(peers, peers + npeers);
  const int64_t* so[2] = {u_send_off, x_send_off};
  const int64_t* si[2] = {u_send_idx, x_send_idx};
  const int64_t* ro[2] = {u_recv_off, x_recv_off};
  const int64_t* ri[2] = {u_recv_idx, x_recv_idx};
  const int w[2] = {u_width, x_width};
  for (int ph = 0; ph < 2; ++ph) {
    Phase& p = c->ph[ph];
    p.width = w[ph];
    p.send_off.assign(npeers + 1, 0);
    p.recv_off.assign(npeers + 1, 0);
    for (int k = 0; k <= npeers && npeers; ++k) {
      p.send_off[k] = so[ph][k];
      p.recv_off[k] = ro[ph][k];
    }
    p.nsend = p.send_off[npeers];
    p.nrecv = p.recv_off[npeers];
    if ((p.nsend && !si[ph]) || (p.nrecv && !ri[ph]))
      return ldg::set_error(2, "missing halo index list", cudaSuccess);
    int rc = up(&p.send_idx, si[ph], p.nsend) | up(&p.recv_idx, ri[ph], p.nrecv) |
             up(&p.send_buf, (const double*)nullptr, p.nsend * p.width) |
             up(&p.recv_buf, (const double*)nullptr, p.nrecv * p.width);
    if (rc) return ldg::set_error(3, "halo plan upload", cudaGetLastError());
  }
  if (npeers && !u_ghost && c->ph[0].nrecv)
    return ldg::set_error(2, "ghost rows need a buffer", cudaSuccess);
  c->planned = true;
  return 0;
}

int ldg_apply_dist(LdgHandle* h, int tangent, const double* u, const double* gproj,
                   const double* bsrc, double* X, double* R, void* stream) {
  NvtxRange nvtx_("ldg_apply_dist");
  Comm* c = comm_of(h);
  if (!c || !c->planned) return ldg::set_error(2, "no halo plan: ldg_set_halo_plan first", cudaSuccess);
  if (!u || !X || !R) return ldg::set_error(2, "bad argument", cudaSuccess);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = run_phase(h, c, 0, u, c->u_ghost, s, tangent, u, gproj, bsrc, X, R);
  if (!rc) rc = run_phase(h, c, 1, X, X, s, tangent, u, gproj, bsrc, X, R);
  return rc;
}

int ldg_comm_destroy(LdgHandle* h) {
  Comm* c = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_comm_m);
    auto it = g_comms.find(h);
    if (it == g_comms.end()) return 0;
    c = it->second;
    g_comms.erase(it);
  }
  cudaStreamSynchronize(c->s_comm);
  free_phase(c->ph[0]);
  free_phase(c->ph[1]);
  if (c->nccl && g_nccl.destroy) g_nccl.destroy(c->nccl);
  cudaEventDestroy(c->ev_pack);
  cudaEventDestroy(c->ev_recv);
  cudaStreamDestroy(c->s_comm);
  delete c;                      // (a local hub is shared by its handles and left to the process)
  return 0;
}

}  // extern "C"
