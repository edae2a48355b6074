// Collectives of one rank: NCCL over NVLink (one process per GPU), or the
// LOOPBACK transport -- `world` virtual ranks driven by host threads of ONE
// process on ONE device, for testing the multi-rank path (a5 exchange, async
// peer puts + version counters, cross-rank detector boards) on a single GPU.
//
// Loopback semantics (SURVEY §4 layer 4): a collective is a host rendezvous of
// the group's threads; every rank first drains its stream, then exchanges
// values through host staging (allreduce / allgather, reduced in rank order)
// or device-to-device copies out of the peer's published buffers (send/recv:
// the peers' buffers are ordinary pointers on the same device).  A second
// rendezvous keeps the published buffers alive until every reader is done.
// Peer "windows" (x storage, detector boards) are the peers' raw pointers, so
// the async kernels store into them exactly as they store over NVLink.
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ctx.h"

namespace ras {

struct LoopGroup {
  int world = 0;
  int refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;                       // a rank timed out: every later rendezvous fails
  std::vector<std::vector<char>> stage;      // per rank: staged host bytes
  std::vector<std::vector<Xfer>> sends;      // per rank: published device send buffers
};

static std::mutex g_groups_mu;
static std::map<std::string, std::shared_ptr<LoopGroup>> g_groups;

static size_t dt_size(ncclDataType_t dt) {
  switch (dt) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 0;
  }
}

ras_status loop_join(ras_ctx* c, const void* key128) {
  std::string key((const char*)key128, 128);
  std::lock_guard<std::mutex> lk(g_groups_mu);
  auto& g = g_groups[key];
  if (!g) {
    g = std::make_shared<LoopGroup>();
    g->world = c->world;
    g->stage.resize(c->world);
    g->sends.resize(c->world);
  }
  if (g->world != c->world) return set_err(c, RAS_EINVAL, "loopback group: world differs between ranks");
  ++g->refs;
  c->loop = g;
  c->loop_key = key;
  return RAS_OK;
}

void loop_leave(ras_ctx* c) {
  if (!c->loop) return;
  std::lock_guard<std::mutex> lk(g_groups_mu);
  if (--c->loop->refs == 0) g_groups.erase(c->loop_key);
  c->loop.reset();
}

// Generation barrier of the group's host threads (timeout: a rank that failed
// never arrives; the others return RAS_ESTATE instead of hanging).
static ras_status loop_barrier(ras_ctx* c) {
  LoopGroup* g = c->loop.get();
  std::unique_lock<std::mutex> lk(g->mu);
  if (g->broken) return set_err(c, RAS_ESTATE, "loopback group broken (a rank failed)");
  const uint64_t my = g->gen;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return RAS_OK;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(600), [&] { return g->gen != my || g->broken; }) || g->broken) {
    g->broken = true;
    g->cv.notify_all();
    return set_err(c, RAS_ESTATE, "loopback rendezvous timed out (a rank never arrived)");
  }
  return RAS_OK;
}

template <class T>
static void reduce_into(std::vector<char>& acc, const std::vector<char>& v, size_t count, bool is_max) {
  T* a = (T*)acc.data();
  const T* b = (const T*)v.data();
  for (size_t i = 0; i < count; ++i) a[i] = is_max ? (a[i] > b[i] ? a[i] : b[i]) : a[i] + b[i];
}

ras_status coll_allreduce(ras_ctx* c, const void* send, void* recv, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                          cudaStream_t s) {
  if (c->world == 1) {
    if (send != recv) RAS_CUDA(c, cudaMemcpyAsync(recv, send, count * dt_size(dt), cudaMemcpyDeviceToDevice, s));
    return RAS_OK;
  }
  if (!c->loop) {
    RAS_NCCL(c, ncclAllReduce(send, recv, count, dt, op, c->nccl, s));
    return RAS_OK;
  }
  if (op != ncclSum && op != ncclMax) return set_err(c, RAS_EINVAL, "loopback allreduce: sum/max only");
  const size_t bytes = count * dt_size(dt);
  LoopGroup* g = c->loop.get();
  g->stage[c->rank].resize(bytes);
  RAS_CUDA(c, cudaMemcpyAsync(g->stage[c->rank].data(), send, bytes, cudaMemcpyDeviceToHost, s));
  RAS_CUDA(c, cudaStreamSynchronize(s));
  TRY(loop_barrier(c));
  std::vector<char> acc = g->stage[0];  // rank order, as written
  for (int r = 1; r < c->world; ++r) {
    const bool mx = op == ncclMax;
    switch (dt) {
      case ncclFloat64: reduce_into<double>(acc, g->stage[r], count, mx); break;
      case ncclInt64: reduce_into<int64_t>(acc, g->stage[r], count, mx); break;
      case ncclInt32: reduce_into<int32_t>(acc, g->stage[r], count, mx); break;
      default: return set_err(c, RAS_EINVAL, "loopback allreduce: unsupported type");
    }
  }
  TRY(loop_barrier(c));  // every rank has read every stage
  RAS_CUDA(c, cudaMemcpyAsync(recv, acc.data(), bytes, cudaMemcpyHostToDevice, s));
  RAS_CUDA(c, cudaStreamSynchronize(s));
  return RAS_OK;
}

ras_status coll_allgather(ras_ctx* c, const void* send, void* recv, size_t count, ncclDataType_t dt, cudaStream_t s) {
  const size_t bytes = count * dt_size(dt);
  if (c->world == 1) {
    if (send != recv) RAS_CUDA(c, cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
    return RAS_OK;
  }
  if (!c->loop) {
    RAS_NCCL(c, ncclAllGather(send, recv, count, dt, c->nccl, s));
    return RAS_OK;
  }
  LoopGroup* g = c->loop.get();
  g->stage[c->rank].resize(bytes);
  RAS_CUDA(c, cudaMemcpyAsync(g->stage[c->rank].data(), send, bytes, cudaMemcpyDeviceToHost, s));
  RAS_CUDA(c, cudaStreamSynchronize(s));
  TRY(loop_barrier(c));
  std::vector<char> all(bytes * c->world);
  for (int r = 0; r < c->world; ++r) std::memcpy(all.data() + r * bytes, g->stage[r].data(), bytes);
  TRY(loop_barrier(c));
  RAS_CUDA(c, cudaMemcpyAsync(recv, all.data(), all.size(), cudaMemcpyHostToDevice, s));
  RAS_CUDA(c, cudaStreamSynchronize(s));
  return RAS_OK;
}

ras_status coll_sendrecv(ras_ctx* c, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, ncclDataType_t dt,
                         cudaStream_t s) {
  if (c->world == 1) return RAS_OK;
  const size_t es = dt_size(dt);
  if (!c->loop) {
    RAS_NCCL(c, ncclGroupStart());
    for (const auto& x : sends)
      if (x.count) RAS_NCCL(c, ncclSend(x.buf, x.count, dt, x.peer, c->nccl, s));
    for (const auto& x : recvs)
      if (x.count) RAS_NCCL(c, ncclRecv(x.buf, x.count, dt, x.peer, c->nccl, s));
    RAS_NCCL(c, ncclGroupEnd());
    return RAS_OK;
  }
  LoopGroup* g = c->loop.get();
  RAS_CUDA(c, cudaStreamSynchronize(s));  // the send buffers are complete (pack kernel done)
  g->sends[c->rank] = sends;
  TRY(loop_barrier(c));
  for (const auto& x : recvs) {
    if (!x.count) continue;
    const Xfer* src = nullptr;
    for (const auto& y : g->sends[x.peer])
      if (y.peer == c->rank) src = &y;
    if (!src || src->count != x.count)
      return set_err(c, RAS_ESTATE, "loopback send/recv: unmatched receive from rank " + std::to_string(x.peer));
    RAS_CUDA(c, cudaMemcpyAsync(x.buf, src->buf, x.count * es, cudaMemcpyDeviceToDevice, s));
  }
  RAS_CUDA(c, cudaStreamSynchronize(s));
  TRY(loop_barrier(c));  // senders may reuse their buffers now
  return RAS_OK;
}

ras_status coll_allreduce_f64(ras_ctx* c, double* v, int n, bool is_max) {
  if (c->world == 1) return RAS_OK;
  std::vector<double> h(v, v + n);
  double* d = (double*)dalloc(c, (size_t)n * 8);
  if (!d) return set_err(c, RAS_ENOMEM, "device allocation failed");
  ras_status st = RAS_OK;
  if (cudaMemcpyAsync(d, h.data(), (size_t)n * 8, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    st = set_err(c, RAS_ECUDA, "cudaMemcpyAsync");
  if (st == RAS_OK) st = coll_allreduce(c, d, d, (size_t)n, ncclFloat64, is_max ? ncclMax : ncclSum, c->stream);
  if (st == RAS_OK && (cudaMemcpyAsync(h.data(), d, (size_t)n * 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                       cudaStreamSynchronize(c->stream) != cudaSuccess))
    st = set_err(c, RAS_ECUDA, "cudaMemcpyAsync");
  dfree(c, d);
  if (st == RAS_OK) std::copy(h.begin(), h.end(), v);
  return st;
}

ras_status coll_barrier(ras_ctx* c) {
  RAS_CUDA(c, cudaDeviceSynchronize());
  if (c->world == 1) return RAS_OK;
  if (c->loop) return loop_barrier(c);
  RAS_NCCL(c, ncclAllReduce(c->d_r2_global, c->d_r2_global, 1, ncclDouble, ncclSum, c->nccl, c->stream));
  RAS_CUDA(c, cudaStreamSynchronize(c->stream));
  return RAS_OK;
}

}  // namespace ras
