// The exchange of ghost-cell data between ranks ("the exchange of the
// cell averages before the reconstruction" and of the reconstruction polynomials
// after it), inside libcwreco.
//
// Transports (chosen by the 128-byte id given to cwreco_set_partition):
//  - NCCL: one communicator per context (ncclCommInitRank), point-to-point
//    ncclSend/ncclRecv per peer inside one ncclGroupStart/End on a library-owned
//    comm stream; over NVLink / NVSwitch between the GPUs of a node.  libnccl is
//    opened with dlopen at cwreco_set_partition time (the process's already
//    loaded NCCL, e.g. torch's, or the system one), so the library itself loads
//    and runs single-rank without NCCL.
//  - loopback: P ranks inside ONE process (one host thread per rank, each with its
//    own context, any device): every peer transfer is one cudaMemcpyAsync from the
//    peer's send buffer into this rank's ghost rows, ordered by CUDA events and a
//    host-side mailbox.  It exercises the whole pack → transfer → boundary-tile
//    path on a single GPU (tests) and is bitwise identical to NCCL (pure copies).
//
// Per exchange (cwreco_halo_exchange / _rows, cwreco_reconstruct_overlap), all on
// the comm stream, ordered after the caller's stream:
//   pack (owned rows requested by each peer, send-list order) → transfer into the
//   ghost rows (directly when the rows are dense, else into a staging buffer and a
//   scatter kernel) → event; the caller's stream (or the boundary tiles) waits on it.
// Ghost rows are ordered by (owner rank, SFC id), so each peer's rows land in one
// contiguous range of the local array.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "devguard.cuh"
#include "internal.hpp"

namespace cwr {

#define HCK(x)                                                                                 \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) fail(CWRECO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

static NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // already in the process
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && api.error.empty()) api.error = std::string("libnccl lacks ") + n;
      return p;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  });
  if (!api.error.empty()) fail(CWRECO_ENCCL, api.error);
  return api;
}

#define NCK(x)                                                                                         \
  do {                                                                                                 \
    ncclResult_t r_ = (x);                                                                             \
    if (r_ != ncclSuccess) fail(CWRECO_ENCCL, std::string(#x) + ": " + nccl().GetErrorString(r_));    \
  } while (0)

// ---------------------------------------------------------------- loopback group
static const char kLoopMagic[8] = {'C', 'W', 'R', 'L', 'O', 'O', 'P', 0};

struct LoopGroup {
  int nranks = 0;
  std::mutex mu;
  std::condition_variable cv;
  // plan exchange: each rank posts its ghost requests (counts per owner, SFC ids)
  std::vector<int64_t> plan_epoch, plan_read;
  std::vector<std::vector<int64_t>> plan_counts, plan_ids;
  // data exchange, per rank: latest epoch posted, its send buffer, row width,
  // send offsets per peer (rows), the event after its pack (parity-indexed)
  struct Post {
    int64_t epoch = -1;
    const double* buf = nullptr;
    int width = 0;
    std::vector<int64_t> send_off;
    cudaEvent_t packed = nullptr;
  };
  std::vector<Post> post;
  // read_epoch[p][r]: last epoch in which reader r finished enqueueing its copies
  // from p's buffer; read_ev[p][r][parity]: event after those copies
  std::vector<std::vector<int64_t>> read_epoch;
  std::vector<std::vector<cudaEvent_t>> read_ev;
  std::vector<bool> joined;
};

static std::mutex g_loop_mu;
static std::map<uint64_t, std::shared_ptr<LoopGroup>> g_loops;
static std::atomic<uint64_t> g_loop_next{1};

// ---------------------------------------------------------------- per-context state
struct HaloState {
  int kind = 0;  // 0 none, 1 NCCL, 2 loopback
  ncclComm_t comm = nullptr;
  std::shared_ptr<LoopGroup> grp;
  uint64_t loop_key = 0;
  cudaStream_t cs = nullptr;  // comm stream
  cudaEvent_t ev_in = nullptr, ev_done = nullptr;
  cudaEvent_t ev_packed[2] = {nullptr, nullptr}, ev_read[2] = {nullptr, nullptr};
  double *sendbuf = nullptr, *recvbuf = nullptr;
  int64_t send_cap = 0, recv_cap = 0;
  int64_t epoch = 0;  // data exchanges done (loopback)
};

static HaloState* hs(const cwreco_ctx* c) { return (HaloState*)c->halo; }

bool halo_has_transport(const cwreco_ctx* c) { return c->halo && hs(c)->kind != 0; }

void halo_unique_id_nccl(uint8_t* id) {
  ncclUniqueId u;
  NCK(nccl().GetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
}

void halo_unique_id_loopback(int nranks, uint8_t* id) {
  if (nranks < 1) fail(CWRECO_EINVAL, "loopback_unique_id: nranks must be >= 1");
  auto g = std::make_shared<LoopGroup>();
  g->nranks = nranks;
  g->plan_epoch.assign(nranks, 0);
  g->plan_read.assign(nranks, 0);
  g->plan_counts.resize(nranks);
  g->plan_ids.resize(nranks);
  g->post.resize(nranks);
  g->read_epoch.assign(nranks, std::vector<int64_t>(nranks, -1));
  g->read_ev.assign(nranks, std::vector<cudaEvent_t>(2 * nranks, nullptr));
  g->joined.assign(nranks, false);
  const uint64_t key = g_loop_next++;
  {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    g_loops[key] = g;
  }
  std::memset(id, 0, 128);
  std::memcpy(id, kLoopMagic, 8);
  std::memcpy(id + 8, &key, 8);
  std::memcpy(id + 16, &nranks, 4);
}

void halo_destroy(cwreco_ctx* c) {
  HaloState* h = hs(c);
  if (!h) return;
  DeviceGuard dg(c->device);
  if (h->cs) cudaStreamSynchronize(h->cs);
  if (h->comm) nccl().CommDestroy(h->comm);
  if (h->grp) {
    std::lock_guard<std::mutex> lk(h->grp->mu);
    h->grp->joined[c->rank] = false;
    h->grp->post[c->rank] = LoopGroup::Post();
  }
  for (cudaEvent_t e : {h->ev_in, h->ev_done, h->ev_packed[0], h->ev_packed[1], h->ev_read[0], h->ev_read[1]})
    if (e) cudaEventDestroy(e);
  if (h->cs) cudaStreamDestroy(h->cs);
  cudaFree(h->sendbuf);
  cudaFree(h->recvbuf);
  delete h;
  c->halo = nullptr;
}

static void make_device_objects(cwreco_ctx* c, HaloState* h) {
  if (c->device < 0) return;  // host-only: plan exchange only
  DeviceGuard dg(c->device);
  HCK(cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&h->ev_in, &h->ev_done, &h->ev_packed[0], &h->ev_packed[1], &h->ev_read[0], &h->ev_read[1]})
    HCK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
}

// cwreco_set_partition(…, id): id == nullptr or nranks == 1 → no transport.
void halo_set_transport(cwreco_ctx* c, const uint8_t* id) {
  halo_destroy(c);
  if (!id || c->nranks == 1) return;
  auto* h = new HaloState();
  c->halo = h;
  try {
    if (std::memcmp(id, kLoopMagic, 8) == 0) {
      uint64_t key;
      int n;
      std::memcpy(&key, id + 8, 8);
      std::memcpy(&n, id + 16, 4);
      std::shared_ptr<LoopGroup> g;
      {
        std::lock_guard<std::mutex> lk(g_loop_mu);
        auto it = g_loops.find(key);
        if (it == g_loops.end()) fail(CWRECO_EINVAL, "set_partition: unknown loopback id");
        g = it->second;
      }
      if (n != c->nranks) fail(CWRECO_EINVAL, "set_partition: loopback id made for another rank count");
      {
        std::lock_guard<std::mutex> lk(g->mu);
        if (g->joined[c->rank]) fail(CWRECO_EINVAL, "set_partition: rank already joined this loopback group");
        g->joined[c->rank] = true;
      }
      h->kind = 2;
      h->grp = g;
      h->loop_key = key;
      make_device_objects(c, h);
    } else {
      if (c->device < 0) fail(CWRECO_ECUDA, "set_partition: an NCCL transport needs a CUDA device");
      DeviceGuard dg(c->device);
      ncclUniqueId u;
      std::memcpy(&u, id, 128);
      NCK(nccl().CommInitRank(&h->comm, c->nranks, u, c->rank));  // collective over the ranks
      h->kind = 1;
      make_device_objects(c, h);
    }
  } catch (...) {
    halo_destroy(c);
    throw;
  }
}

// ---------------------------------------------------------------- plan exchange
// After the stencils (collective over the ranks): every rank tells each owner which
// of its cells it needs; the owner installs them as its send lists.
void halo_plan_exchange(cwreco_ctx* c) {
  HaloState* h = hs(c);
  if (!h || h->kind == 0) return;
  const int P = c->nranks, me = c->rank;
  const std::vector<int64_t>& rc = c->ghost_counts;
  std::vector<int64_t> rid(c->local2global.begin() + c->n_owned, c->local2global.end());
  std::vector<int64_t> sc(P, 0), sid;
  if (h->kind == 2) {
    LoopGroup& g = *h->grp;
    std::unique_lock<std::mutex> lk(g.mu);
    g.plan_counts[me] = rc;
    g.plan_ids[me] = rid;
    const int64_t ep = ++g.plan_epoch[me];
    g.cv.notify_all();
    g.cv.wait(lk, [&] {
      for (int p = 0; p < P; ++p)
        if (g.plan_epoch[p] < ep) return false;
      return true;
    });
    for (int p = 0; p < P; ++p) {
      int64_t off = 0;
      for (int q = 0; q < me; ++q) off += g.plan_counts[p][q];
      sc[p] = g.plan_counts[p][me];
      sid.insert(sid.end(), g.plan_ids[p].begin() + off, g.plan_ids[p].begin() + off + sc[p]);
    }
    // nobody may post the next plan before every rank has read this one
    g.plan_read[me] = ep;
    g.cv.notify_all();
    g.cv.wait(lk, [&] {
      for (int p = 0; p < P; ++p)
        if (g.plan_read[p] < ep) return false;
      return true;
    });
  } else {
    NcclApi& api = nccl();
    DeviceGuard dg(c->device);
    int64_t *d_rc = nullptr, *d_sc = nullptr, *d_rid = nullptr, *d_sid = nullptr;
    auto cleanup = [&] {
      cudaFree(d_rc);
      cudaFree(d_sc);
      cudaFree(d_rid);
      cudaFree(d_sid);
    };
    try {
      HCK(cudaMalloc(&d_rc, P * 8));
      HCK(cudaMalloc(&d_sc, P * 8));
      HCK(cudaMemcpy(d_rc, rc.data(), P * 8, cudaMemcpyHostToDevice));
      HCK(cudaMemset(d_sc, 0, P * 8));
      NCK(api.GroupStart());
      for (int p = 0; p < P; ++p) {
        if (p == me) continue;
        NCK(api.Send(d_rc + p, 1, ncclInt64, p, h->comm, h->cs));
        NCK(api.Recv(d_sc + p, 1, ncclInt64, p, h->comm, h->cs));
      }
      NCK(api.GroupEnd());
      HCK(cudaStreamSynchronize(h->cs));
      HCK(cudaMemcpy(sc.data(), d_sc, P * 8, cudaMemcpyDeviceToHost));
      int64_t ns = 0;
      for (int p = 0; p < P; ++p) ns += sc[p];
      HCK(cudaMalloc(&d_rid, std::max<int64_t>(1, (int64_t)rid.size()) * 8));
      HCK(cudaMalloc(&d_sid, std::max<int64_t>(1, ns) * 8));
      if (!rid.empty()) HCK(cudaMemcpy(d_rid, rid.data(), rid.size() * 8, cudaMemcpyHostToDevice));
      NCK(api.GroupStart());
      int64_t ro = 0, so = 0;
      for (int p = 0; p < P; ++p) {
        if (rc[p] > 0) NCK(api.Send(d_rid + ro, (size_t)rc[p], ncclInt64, p, h->comm, h->cs));
        if (sc[p] > 0) NCK(api.Recv(d_sid + so, (size_t)sc[p], ncclInt64, p, h->comm, h->cs));
        ro += rc[p];
        so += sc[p];
      }
      NCK(api.GroupEnd());
      HCK(cudaStreamSynchronize(h->cs));
      sid.resize(ns);
      if (ns) HCK(cudaMemcpy(sid.data(), d_sid, ns * 8, cudaMemcpyDeviceToHost));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  }
  install_send_lists(c, sc.data(), sid.data());
}

// ---------------------------------------------------------------- data exchange
__global__ void k_halo_unpack(const double* __restrict__ buf, int64_t n, int W, double* __restrict__ rows,
                              int64_t rs, int64_t es) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= n * W) return;
  const int64_t k = gid / W;
  const int e = int(gid % W);
  rows[k * rs + e * es] = buf[gid];
}

static void grow(double*& p, int64_t& cap, int64_t n) {
  if (cap >= n) return;
  cudaFree(p);
  p = nullptr;
  cap = 0;
  if (cudaMalloc(&p, std::max<int64_t>(1, n) * 8) != cudaSuccess) {
    cudaGetLastError();
    fail(CWRECO_ENOMEM, "halo exchange: buffer allocation failed");
  }
  cap = n;
}

// Enqueue the exchange of W-wide rows (element (k, e) at rows[k·rs + e·es]) on the
// comm stream after the work already on `stream`; records h->ev_done when the ghost
// rows are complete.  The caller makes its stream (or the boundary tiles) wait.
void halo_exchange_begin(cwreco_ctx* c, double* rows, int64_t rs, int64_t es, int W, cudaStream_t stream) {
  HaloState* h = hs(c);
  if (!h || h->kind == 0) fail(CWRECO_ESTATE, "halo exchange: no transport (cwreco_set_partition with an id)");
  if (c->device < 0 || !h->cs) fail(CWRECO_ECUDA, "halo exchange: host-only context (no CUDA device)");
  DeviceGuard dg(c->device);
  const int P = c->nranks, me = c->rank;
  const int64_t n_send = (int64_t)c->send_local.size(), n_ghost = c->n_ghost;
  const bool dense = es == 1 && rs == W;
  grow(h->sendbuf, h->send_cap, n_send * W);
  if (!dense) grow(h->recvbuf, h->recv_cap, n_ghost * W);
  double* dst = dense ? rows + c->n_owned * rs : h->recvbuf;
  std::vector<int64_t> send_off(P + 1, 0), recv_off(P + 1, 0);
  for (int p = 0; p < P; ++p) {
    send_off[p + 1] = send_off[p] + c->send_counts[p];
    recv_off[p + 1] = recv_off[p] + c->ghost_counts[p];
  }
  HCK(cudaEventRecord(h->ev_in, stream));
  HCK(cudaStreamWaitEvent(h->cs, h->ev_in, 0));
  const int64_t ep = h->epoch++;
  const int par = int(ep & 1);
  if (h->kind == 2 && ep > 0) {
    // every peer that read our previous buffer (epoch ep−1) must be done with it
    // before it is repacked: wait for their posts, then for their copy events
    LoopGroup& g = *h->grp;
    std::vector<cudaEvent_t> wait;
    {
      std::unique_lock<std::mutex> lk(g.mu);
      g.cv.wait(lk, [&] {
        for (int r = 0; r < P; ++r)
          if (r != me && c->send_counts[r] > 0 && g.read_epoch[me][r] < ep - 1) return false;
        return true;
      });
      for (int r = 0; r < P; ++r)
        if (r != me && c->send_counts[r] > 0) wait.push_back(g.read_ev[me][2 * r + ((ep - 1) & 1)]);
    }
    for (cudaEvent_t e : wait) HCK(cudaStreamWaitEvent(h->cs, e, 0));
  }
  if (n_send > 0) dev_halo_pack_rows(c, rows, rs, es, W, h->sendbuf, h->cs);
  if (h->kind == 1) {
    NcclApi& api = nccl();
    NCK(api.GroupStart());
    for (int p = 0; p < P; ++p) {
      const int64_t ns = c->send_counts[p], nr = c->ghost_counts[p];
      if (ns > 0) NCK(api.Send(h->sendbuf + send_off[p] * W, (size_t)(ns * W), ncclFloat64, p, h->comm, h->cs));
      if (nr > 0) NCK(api.Recv(dst + recv_off[p] * W, (size_t)(nr * W), ncclFloat64, p, h->comm, h->cs));
    }
    NCK(api.GroupEnd());
  } else {
    LoopGroup& g = *h->grp;
    HCK(cudaEventRecord(h->ev_packed[par], h->cs));
    {
      std::lock_guard<std::mutex> lk(g.mu);
      LoopGroup::Post& po = g.post[me];
      po.epoch = ep;
      po.buf = h->sendbuf;
      po.width = W;
      po.send_off = send_off;
      po.packed = h->ev_packed[par];
      g.cv.notify_all();
    }
    for (int p = 0; p < P; ++p) {
      const int64_t nr = c->ghost_counts[p];
      if (nr == 0 || p == me) continue;
      const double* src;
      cudaEvent_t pk;
      {
        std::unique_lock<std::mutex> lk(g.mu);
        g.cv.wait(lk, [&] { return g.post[p].epoch >= ep; });
        if (g.post[p].epoch != ep || g.post[p].width != W)
          fail(CWRECO_ESTATE, "loopback halo exchange: ranks out of step (every rank must exchange the same rows)");
        src = g.post[p].buf + g.post[p].send_off[me] * W;
        if (g.post[p].send_off[me + 1] - g.post[p].send_off[me] != nr)
          fail(CWRECO_ESTATE, "loopback halo exchange: peer send list does not match this rank's ghosts");
        pk = g.post[p].packed;
      }
      HCK(cudaStreamWaitEvent(h->cs, pk, 0));
      HCK(cudaMemcpyAsync(dst + recv_off[p] * W, src, nr * W * 8, cudaMemcpyDefault, h->cs));
    }
    HCK(cudaEventRecord(h->ev_read[par], h->cs));
    {
      std::lock_guard<std::mutex> lk(g.mu);
      for (int p = 0; p < P; ++p) {
        if (p == me || c->ghost_counts[p] == 0) continue;
        g.read_ev[p][2 * me + par] = h->ev_read[par];
        g.read_epoch[p][me] = ep;
      }
      g.cv.notify_all();
    }
  }
  if (!dense && n_ghost > 0) {
    const int64_t th = n_ghost * W;
    k_halo_unpack<<<(unsigned)((th + 255) / 256), 256, 0, h->cs>>>(h->recvbuf, n_ghost, W, rows + c->n_owned * rs, rs,
                                                                   es);
    HCK(cudaGetLastError());
  }
  HCK(cudaEventRecord(h->ev_done, h->cs));
}

void halo_exchange(cwreco_ctx* c, double* rows, int64_t rs, int64_t es, int W, void* stream) {
  halo_exchange_begin(c, rows, rs, es, W, (cudaStream_t)stream);
  DeviceGuard dg(c->device);
  HCK(cudaStreamWaitEvent((cudaStream_t)stream, hs(c)->ev_done, 0));
}

// One overlapped pass (§8(b) overlap_halo): exchange on the comm stream, interior
// tiles on `stream` concurrently (they read no ghost row), then the boundary tiles
// after the exchange event.
void halo_reconstruct_overlap(cwreco_ctx* c, double* avgs, int64_t acs, int64_t avs, double* coeffs, int64_t ccs,
                              int64_t cvs, void* stream) {
  halo_exchange_begin(c, avgs, acs, avs, c->V, (cudaStream_t)stream);
  dev_reconstruct(c, avgs, acs, avs, coeffs, ccs, cvs, CWRECO_PART_INTERIOR, stream);
  {
    DeviceGuard dg(c->device);
    HCK(cudaStreamWaitEvent((cudaStream_t)stream, hs(c)->ev_done, 0));
  }
  dev_reconstruct(c, avgs, acs, avs, coeffs, ccs, cvs, CWRECO_PART_BOUNDARY, stream);
}

}  // namespace cwr
