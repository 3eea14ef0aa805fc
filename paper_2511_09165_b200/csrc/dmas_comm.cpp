// Multi-GPU exchange of direction-sharded plans: NCCL resolved at run time, the gather schedule.
// See dmas_comm.h.  NCCL's types come from its header; no link-time dependency.

#include "dmas_comm.h"

#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include <cuda.h>
#include <nccl.h>

namespace dmas {
namespace comm {

void shard_range(int64_t n, int32_t n_ranks, int32_t rank, int64_t* g0, int64_t* g1) {
  const int64_t base = n / n_ranks, extra = n % n_ranks;
  *g0 = rank * base + std::min<int64_t>(rank, extra);
  *g1 = *g0 + base + (rank < extra ? 1 : 0);
}

std::vector<dmas_xfer> gather_schedule(int64_t n_dirs, int32_t n_ranks, int32_t rank, int32_t root, int32_t n_frames,
                                       int64_t row_elems) {
  std::vector<dmas_xfer> xs;
  int64_t my0, my1;
  shard_range(n_dirs, n_ranks, rank, &my0, &my1);
  const int64_t my_n = my1 - my0;
  for (int32_t f = 0; f < n_frames; ++f) {
    for (int32_t r = 0; r < n_ranks; ++r) {
      int64_t g0, g1;
      shard_range(n_dirs, n_ranks, r, &g0, &g1);
      if (g1 == g0) continue;                                   // more ranks than directions
      dmas_xfer x{};
      x.frame = f;
      x.count = (g1 - g0) * row_elems;
      if (rank == root && r == root) {
        x.kind = DMAS_XFER_COPY;
        x.peer = root;
        x.src_elem = (int64_t)f * my_n * row_elems;
        x.dst_elem = ((int64_t)f * n_dirs + g0) * row_elems;
      } else if (rank == root) {
        x.kind = DMAS_XFER_RECV;
        x.peer = r;
        x.src_elem = -1;
        x.dst_elem = ((int64_t)f * n_dirs + g0) * row_elems;
      } else if (r == rank) {
        x.kind = DMAS_XFER_SEND;
        x.peer = root;
        x.src_elem = (int64_t)f * my_n * row_elems;
        x.dst_elem = -1;
      } else {
        continue;
      }
      xs.push_back(x);
    }
  }
  return xs;
}

// ---------------------------------------------------------------------------------- NCCL (dlopen)
namespace {

struct Api {
  bool loaded = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    // the NCCL the process already has (torch's) first, so one process never holds two NCCLs
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    bool ok = true;
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) ok = false;
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.CommAbort = reinterpret_cast<decltype(a.CommAbort)>(sym("ncclCommAbort"));
    a.CommGetAsyncError = reinterpret_cast<decltype(a.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    if (!ok) {
      a.why = "libnccl.so.2 lacks a required symbol";
      return;
    }
    a.loaded = true;
  });
  return a;
}

dmas_status nccl_fail(ncclResult_t r, const char* what, std::string& err) {
  const Api& a = api();
  err = std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "NCCL error");
  return DMAS_ERR_NCCL;
}

#define NCCL_TRY(expr, what)                                   \
  do {                                                         \
    ncclResult_t r_ = (expr);                                  \
    if (r_ != ncclSuccess) return nccl_fail(r_, what, err);    \
  } while (0)

}  // namespace

// ---------------------------------------------------------------------------------- loopback
// In-process test transport (comm_id starting with "DMASLOOP"): the ranks are plans of ONE
// process -- threads, on any devices -- and the exchange runs as device-to-device copies ordered
// by CUDA events, with NCCL's semantics: operations match in issue order per peer pair, a
// broadcast / send completes on the sender's stream only once the receivers' copies are done
// (so the sender may then reuse its buffer).  Every rank thread blocks (host side) until its
// peers have enqueued their side of an operation, as NCCL's ranks progress together.  It lets
// the multi-rank exchange of the runtime (chunk agreement, staging reuse, gather assembly, host
// path) run on one GPU without two ranks ever waiting on each other inside a kernel.
namespace {
struct LoopMsg {
  const void* src = nullptr;
  size_t bytes = 0;
  cudaEvent_t ready = nullptr;            // recorded on the sender's stream after its data is ready
  std::vector<cudaEvent_t> done;          // recorded on each receiver's stream after its copy
};
struct LoopGroup {
  std::mutex mu;
  std::condition_variable cv;
  int32_t n_ranks = 0;
  int ar_count = 0;
  int64_t ar_gen = 0, ar_acc = 0, ar_result = 0;
  std::map<int64_t, LoopMsg> bcast;                                   // by broadcast sequence
  std::map<int64_t, void*> ptrs;                                      // fused gather: root buffers
  std::map<int64_t, std::vector<cudaEvent_t>> bars;                   // root barriers: ranks' events
  std::map<std::tuple<int32_t, int32_t, int64_t>, LoopMsg> p2p;       // (src, dst, sequence)
};
std::mutex g_loop_mu;
std::map<std::string, std::weak_ptr<LoopGroup>> g_loop_groups;
constexpr char kLoopMagic[8] = {'D', 'M', 'A', 'S', 'L', 'O', 'O', 'P'};
}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  std::shared_ptr<LoopGroup> loop;        // loopback transport (tests), else NCCL
  int32_t n_ranks = 1, rank = 0;
  int64_t bseq = 0;                       // loopback: broadcasts issued
  std::map<int32_t, int64_t> sseq, rseq;  // loopback: sends to / receives from each peer
  int64_t mseq = 0, barseq = 0;           // loopback: root-buffer exchanges / root barriers
  void* xbuf = nullptr;                   // NCCL: small device buffer for control words
  std::map<std::string, void*> ipc_open;  // NCCL: root allocations opened by CUDA IPC (non-root ranks)
};

namespace {
dmas_status cuda_fail(cudaError_t e, const char* what, std::string& err) {
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return DMAS_ERR_CUDA;
}
#define LOOP_TRY(expr, what)                                    \
  do {                                                          \
    cudaError_t e_ = (expr);                                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, what, err);     \
  } while (0)

// sender side: publish `src` (ready once `st` reaches this point), then make `st` wait until
// every one of `n_recv` receivers has copied it
dmas_status loop_publish_and_wait(LoopGroup& g, std::unique_lock<std::mutex>& lk, LoopMsg& m, size_t n_recv,
                                  cudaStream_t st, std::string& err) {
  g.cv.notify_all();
  g.cv.wait(lk, [&] { return m.done.size() >= n_recv; });
  for (cudaEvent_t e : m.done) {
    LOOP_TRY(cudaStreamWaitEvent(st, e, 0), "loopback: wait for receivers");
    cudaEventDestroy(e);
  }
  cudaEventDestroy(m.ready);
  return DMAS_OK;
}
// receiver side: copy the published message into `dst` on `st`, then report done
dmas_status loop_receive(LoopGroup& g, LoopMsg& m, void* dst, size_t bytes, cudaStream_t st, std::string& err) {
  if (m.bytes != bytes) {
    err = "loopback: message size mismatch (" + std::to_string(m.bytes) + " vs " + std::to_string(bytes) + ")";
    return DMAS_ERR_NCCL;
  }
  LOOP_TRY(cudaStreamWaitEvent(st, m.ready, 0), "loopback: wait for sender");
  if (dst != m.src) LOOP_TRY(cudaMemcpyAsync(dst, m.src, bytes, cudaMemcpyDefault, st), "loopback: copy");
  cudaEvent_t d = nullptr;
  LOOP_TRY(cudaEventCreateWithFlags(&d, cudaEventDisableTiming), "loopback: event");
  LOOP_TRY(cudaEventRecord(d, st), "loopback: record");
  m.done.push_back(d);
  g.cv.notify_all();
  return DMAS_OK;
}
}  // namespace

dmas_status unique_id(uint8_t out[DMAS_COMM_ID_BYTES], std::string& err) {
  static_assert(DMAS_COMM_ID_BYTES == NCCL_UNIQUE_ID_BYTES, "comm id size");
  const Api& a = api();
  if (!a.loaded) {
    err = a.why;
    return DMAS_ERR_NCCL;
  }
  ncclUniqueId id;
  NCCL_TRY(a.GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, DMAS_COMM_ID_BYTES);
  return DMAS_OK;
}

dmas_status create(const uint8_t id[DMAS_COMM_ID_BYTES], int32_t n_ranks, int32_t rank, Comm** out,
                   std::string& err) {
  if (std::memcmp(id, kLoopMagic, sizeof(kLoopMagic)) == 0) {
    const std::string key(reinterpret_cast<const char*>(id), DMAS_COMM_ID_BYTES);
    std::lock_guard<std::mutex> lk(g_loop_mu);
    std::shared_ptr<LoopGroup> g = g_loop_groups[key].lock();
    if (!g) {
      g = std::make_shared<LoopGroup>();
      g->n_ranks = n_ranks;
      g_loop_groups[key] = g;
    }
    if (g->n_ranks != n_ranks) {
      err = "loopback: ranks disagree on n_ranks";
      return DMAS_ERR_NCCL;
    }
    auto* c = new Comm();
    c->loop = g;
    c->n_ranks = n_ranks;
    c->rank = rank;
    *out = c;
    return DMAS_OK;
  }
  const Api& a = api();
  if (!a.loaded) {
    err = a.why;
    return DMAS_ERR_NCCL;
  }
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, DMAS_COMM_ID_BYTES);
  auto* c = new Comm();
  c->n_ranks = n_ranks;
  c->rank = rank;
  const ncclResult_t r = a.CommInitRank(&c->comm, n_ranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank", err);
  }
  if (cudaMalloc(&c->xbuf, 256) != cudaSuccess) {
    destroy(c);
    err = "cudaMalloc (control words)";
    return DMAS_ERR_OOM;
  }
  *out = c;
  return DMAS_OK;
}

namespace {
// base address of the allocation holding `p` (driver API through the runtime's entry point)
bool allocation_base(void* p, void** base) {
  typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<RangeFn>(f);
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) return false;
  *base = reinterpret_cast<void*>(b);
  return true;
}
}  // namespace

dmas_status map_root_buffer(Comm* c, void* root_ptr, int32_t root, void** mapped, cudaStream_t st,
                            std::string& err) {
  const bool is_root = c->rank == root;
  if (c->loop) {
    LoopGroup& g = *c->loop;
    const int64_t seq = c->mseq++;
    std::unique_lock<std::mutex> lk(g.mu);
    if (is_root) {
      g.ptrs[seq] = root_ptr;
      g.cv.notify_all();
      *mapped = root_ptr;
      return DMAS_OK;
    }
    g.cv.wait(lk, [&] { return g.ptrs.count(seq) > 0; });
    *mapped = g.ptrs[seq];
    return DMAS_OK;
  }
  // NCCL: the root exports its allocation (IPC handle + offset), every rank receives it
  struct Msg {
    cudaIpcMemHandle_t h;
    int64_t offset;
    int64_t ok;
  } m{};
  static_assert(sizeof(Msg) <= 256, "control words");
  if (is_root) {
    void* base = nullptr;
    m.ok = allocation_base(root_ptr, &base) && cudaIpcGetMemHandle(&m.h, base) == cudaSuccess;
    m.offset = m.ok ? (int64_t)((char*)root_ptr - (char*)base) : 0;
    LOOP_TRY(cudaMemcpyAsync(c->xbuf, &m, sizeof(Msg), cudaMemcpyHostToDevice, st), "fused gather: handle");
  }
  NCCL_TRY(api().Broadcast(c->xbuf, c->xbuf, sizeof(Msg), ncclChar, root, c->comm, st), "ncclBroadcast (handle)");
  LOOP_TRY(cudaMemcpyAsync(&m, c->xbuf, sizeof(Msg), cudaMemcpyDeviceToHost, st), "fused gather: handle");
  LOOP_TRY(cudaStreamSynchronize(st), "fused gather: handle");
  if (!m.ok) {
    err = "fused gather: the root's output buffer cannot be exported by CUDA IPC";
    return DMAS_ERR_NCCL;
  }
  if (is_root) {
    *mapped = root_ptr;
    return DMAS_OK;
  }
  const std::string key(reinterpret_cast<const char*>(&m.h), sizeof(m.h));
  auto it = c->ipc_open.find(key);
  if (it == c->ipc_open.end()) {
    void* b = nullptr;
    LOOP_TRY(cudaIpcOpenMemHandle(&b, m.h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    it = c->ipc_open.emplace(key, b).first;
  }
  *mapped = (char*)it->second + m.offset;
  return DMAS_OK;
}

dmas_status root_barrier(Comm* c, int32_t root, cudaStream_t st, std::string& err) {
  if (c->loop) {
    LoopGroup& g = *c->loop;
    const int64_t seq = c->barseq++;
    std::unique_lock<std::mutex> lk(g.mu);
    if (c->rank != root) {
      cudaEvent_t e = nullptr;
      LOOP_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "loopback: event");
      LOOP_TRY(cudaEventRecord(e, st), "loopback: record");
      g.bars[seq].push_back(e);
      g.cv.notify_all();
      return DMAS_OK;
    }
    g.cv.wait(lk, [&] { return (int)g.bars[seq].size() >= c->n_ranks - 1; });
    for (cudaEvent_t e : g.bars[seq]) {
      LOOP_TRY(cudaStreamWaitEvent(st, e, 0), "loopback: barrier");
      cudaEventDestroy(e);
    }
    g.bars.erase(seq);
    return DMAS_OK;
  }
  NCCL_TRY(api().AllReduce(c->xbuf, c->xbuf, 1, ncclInt32, ncclSum, c->comm, st), "ncclAllReduce (barrier)");
  return DMAS_OK;
}

void destroy(Comm* c) {
  if (!c) return;
  if (c->loop) {
    delete c;
    return;
  }
  for (auto& kv : c->ipc_open) cudaIpcCloseMemHandle(kv.second);
  cudaFree(c->xbuf);
  const Api& a = api();
  if (c->comm && a.loaded) {
    ncclResult_t ae = ncclSuccess;
    a.CommGetAsyncError(c->comm, &ae);
    if (ae != ncclSuccess) a.CommAbort(c->comm);
    else a.CommDestroy(c->comm);
  }
  delete c;
}

dmas_status broadcast(Comm* c, float* buf, size_t count, int32_t root, cudaStream_t st, std::string& err) {
  if (c->loop) {
    LoopGroup& g = *c->loop;
    const int64_t seq = c->bseq++;
    const size_t bytes = count * sizeof(float);
    std::unique_lock<std::mutex> lk(g.mu);
    if (c->rank == root) {
      LoopMsg& m = g.bcast[seq];
      m.src = buf;
      m.bytes = bytes;
      LOOP_TRY(cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming), "loopback: event");
      LOOP_TRY(cudaEventRecord(m.ready, st), "loopback: record");
      dmas_status rc = loop_publish_and_wait(g, lk, m, (size_t)(c->n_ranks - 1), st, err);
      g.bcast.erase(seq);
      return rc;
    }
    g.cv.wait(lk, [&] { auto it = g.bcast.find(seq); return it != g.bcast.end() && it->second.ready; });
    return loop_receive(g, g.bcast[seq], buf, bytes, st, err);
  }
  NCCL_TRY(api().Broadcast(buf, buf, count, ncclFloat32, root, c->comm, st), "ncclBroadcast");
  return DMAS_OK;
}

dmas_status allreduce_min(Comm* c, int64_t* v, cudaStream_t st, std::string& err) {
  if (c->loop) {
    LoopGroup& g = *c->loop;
    std::unique_lock<std::mutex> lk(g.mu);
    const int64_t gen = g.ar_gen;
    g.ar_acc = g.ar_count == 0 ? *v : std::min(g.ar_acc, *v);
    if (++g.ar_count == g.n_ranks) {
      g.ar_result = g.ar_acc;
      g.ar_count = 0;
      ++g.ar_gen;
      g.cv.notify_all();
    } else {
      g.cv.wait(lk, [&] { return g.ar_gen != gen; });
    }
    *v = g.ar_result;
    return DMAS_OK;
  }
  int64_t* d = nullptr;
  if (cudaMalloc(&d, sizeof(int64_t)) != cudaSuccess) {
    err = "cudaMalloc (allreduce scratch)";
    return DMAS_ERR_OOM;
  }
  dmas_status rc = DMAS_OK;
  if (cudaMemcpyAsync(d, v, sizeof(int64_t), cudaMemcpyHostToDevice, st) != cudaSuccess) rc = DMAS_ERR_CUDA;
  if (rc == DMAS_OK) {
    const ncclResult_t r = api().AllReduce(d, d, 1, ncclInt64, ncclMin, c->comm, st);
    if (r != ncclSuccess) rc = nccl_fail(r, "ncclAllReduce", err);
  }
  if (rc == DMAS_OK && (cudaMemcpyAsync(v, d, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                        cudaStreamSynchronize(st) != cudaSuccess)) {
    err = "allreduce copy-back";
    rc = DMAS_ERR_CUDA;
  }
  cudaFree(d);
  return rc;
}

dmas_status run_gather(Comm* c, const std::vector<dmas_xfer>& xs, const float* shard, float* dst, cudaStream_t st,
                       std::string& err) {
  const Api& a = api();
  // local rows first (plain device copies), then every send / recv of the chunk in one NCCL group
  for (const dmas_xfer& x : xs)
    if (x.kind == DMAS_XFER_COPY) {
      const cudaError_t e = cudaMemcpyAsync(dst + x.dst_elem, shard + x.src_elem, (size_t)x.count * sizeof(float),
                                            cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) {
        err = std::string("gather copy: ") + cudaGetErrorString(e);
        return DMAS_ERR_CUDA;
      }
    }
  bool any = false;
  for (const dmas_xfer& x : xs) any |= x.kind != DMAS_XFER_COPY;
  if (!any) return DMAS_OK;
  if (c->loop) {
    LoopGroup& g = *c->loop;
    for (const dmas_xfer& x : xs) {
      const size_t bytes = (size_t)x.count * sizeof(float);
      std::unique_lock<std::mutex> lk(g.mu);
      if (x.kind == DMAS_XFER_SEND) {
        const auto key = std::make_tuple(c->rank, x.peer, c->sseq[x.peer]++);
        LoopMsg& m = g.p2p[key];
        m.src = shard + x.src_elem;
        m.bytes = bytes;
        LOOP_TRY(cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming), "loopback: event");
        LOOP_TRY(cudaEventRecord(m.ready, st), "loopback: record");
        dmas_status rc = loop_publish_and_wait(g, lk, m, 1, st, err);
        g.p2p.erase(key);
        if (rc != DMAS_OK) return rc;
      } else if (x.kind == DMAS_XFER_RECV) {
        const auto key = std::make_tuple(x.peer, c->rank, c->rseq[x.peer]++);
        g.cv.wait(lk, [&] { auto it = g.p2p.find(key); return it != g.p2p.end() && it->second.ready; });
        dmas_status rc = loop_receive(g, g.p2p[key], dst + x.dst_elem, bytes, st, err);
        if (rc != DMAS_OK) return rc;
      }
    }
    return DMAS_OK;
  }
  NCCL_TRY(a.GroupStart(), "ncclGroupStart");
  for (const dmas_xfer& x : xs) {
    ncclResult_t r = ncclSuccess;
    if (x.kind == DMAS_XFER_SEND) r = a.Send(shard + x.src_elem, (size_t)x.count, ncclFloat32, x.peer, c->comm, st);
    else if (x.kind == DMAS_XFER_RECV) r = a.Recv(dst + x.dst_elem, (size_t)x.count, ncclFloat32, x.peer, c->comm, st);
    if (r != ncclSuccess) {
      a.GroupEnd();
      return nccl_fail(r, x.kind == DMAS_XFER_SEND ? "ncclSend" : "ncclRecv", err);
    }
  }
  NCCL_TRY(a.GroupEnd(), "ncclGroupEnd");
  return DMAS_OK;
}

}  // namespace comm
}  // namespace dmas
