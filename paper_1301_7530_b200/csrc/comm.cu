// Row-sharded multi-GPU plumbing: NCCL (loaded with dlopen, so librcg.so
// has no hard NCCL dependency) for the halo exchange of SpMV ghost entries
// and the packed fp64 allreduces of the per-iteration reduction slots
// (SURVEY.md §8(e)).  One process per GPU; every rank holds a contiguous row
// slab, and the ghost values it reads live in a region appended after its
// n_local entries of every SpMV-input column (W[:, j], C[:, c], x0).
#include "rcg_internal.cuh"
#include "comm.cuh"

#include <dlfcn.h>
#include <algorithm>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <vector>

namespace rcg {

// minimal NCCL ABI (nccl.h 2.x): types and the entry points we call
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { kNcclFloat64 = 8, kNcclSum = 0 };

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

// Single-process loopback transport (validation of the sharded path on one
// GPU): ranks are host threads with their own streams on the same device.
// Collectives exchange data with device copies ordered by CUDA events;
// a host barrier per collective guarantees every event a stream waits on has
// already been recorded, so all dependencies point to enqueued work (no
// kernel ever spins on another rank).
struct LoopGroup {
  int nranks = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  // per rank, two slot sets (round parity) for allreduce / halo staging
  std::vector<double*> slot[2];
  std::vector<size_t> slot_cap[2];
  std::vector<cudaEvent_t> ready[2];     // slot written (recorded by its owner)
  std::vector<cudaEvent_t> consumed[2];  // owner's consumption of everyone's slots done
  std::vector<const rcg_halo*> halo;     // halo plan of each rank (current exchange)
  std::vector<double*> send_buf;         // each rank's packed send buffer (current exchange)
  long long round[64] = {0};
  void barrier() {
    std::unique_lock<std::mutex> l(mu);
    const long long gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(l, [&] { return generation != gen; });
    }
  }
};

struct Comm {
  Nccl api;
  ncclComm_t comm = nullptr;
  int nranks = 1;
  int rank = 0;
  LoopGroup* loop = nullptr;
};

static int load_nccl(const char* path, Nccl* n, std::string* err) {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch already loaded
  if (!h && path && *path) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    *err = std::string("cannot load NCCL: ") + dlerror();
    return RCG_ERR_CUDA;
  }
  n->h = h;
#define RCG_SYM(field, name)                                  \
  *(void**)(&n->field) = dlsym(h, name);                      \
  if (!n->field) {                                            \
    *err = std::string("NCCL symbol missing: ") + name;       \
    return RCG_ERR_CUDA;                                      \
  }
  RCG_SYM(getUniqueId, "ncclGetUniqueId");
  RCG_SYM(commInitRank, "ncclCommInitRank");
  RCG_SYM(commDestroy, "ncclCommDestroy");
  RCG_SYM(allReduce, "ncclAllReduce");
  RCG_SYM(send, "ncclSend");
  RCG_SYM(recv, "ncclRecv");
  RCG_SYM(groupStart, "ncclGroupStart");
  RCG_SYM(groupEnd, "ncclGroupEnd");
  RCG_SYM(errStr, "ncclGetErrorString");
#undef RCG_SYM
  return RCG_OK;
}

#define RCG_NCCL(ctx, call)                                                                      \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != 0)                                                                                 \
      return set_error((ctx), RCG_ERR_CUDA, "%s: %s", #call, (ctx)->comm->api.errStr(r_));        \
  } while (0)

int comm_ranks(const Ctx* c) { return c->comm ? c->comm->nranks : 1; }

__global__ void sum_slots_kernel(double* out, double* const* slots, int nranks, size_t count) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += slots[r][i];   // rank order: identical bits on every rank
    out[i] = s;
  }
}

static int loop_allreduce(Ctx* c, double* buf, size_t count) {
  LoopGroup* g = c->comm->loop;
  const int me = c->comm->rank, R = g->nranks;
  const int par = (int)(g->round[me] & 1);
  ++g->round[me];
  // my slot of this parity was last read two rounds ago: wait for every rank's consumption
  for (int q = 0; q < R; ++q) RCG_CUDA(c, cudaStreamWaitEvent(c->stream, g->consumed[par][q], 0));
  if (g->slot_cap[par][me] < count) {
    // grow (all ranks are past the previous use of this parity, see the wait above)
    RCG_CUDA(c, cudaStreamSynchronize(c->stream));
    if (g->slot[par][me]) cudaFree(g->slot[par][me]);
    RCG_CUDA(c, cudaMalloc(&g->slot[par][me], std::max<size_t>(count, 4096) * sizeof(double)));
    g->slot_cap[par][me] = std::max<size_t>(count, 4096);
  }
  RCG_CUDA(c, cudaMemcpyAsync(g->slot[par][me], buf, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  RCG_CUDA(c, cudaEventRecord(g->ready[par][me], c->stream));
  g->barrier();  // every rank's slot copy + event is enqueued
  for (int q = 0; q < R; ++q)
    if (q != me) RCG_CUDA(c, cudaStreamWaitEvent(c->stream, g->ready[par][q], 0));
  double** dptrs = nullptr;
  RCG_CUDA(c, cudaMallocAsync((void**)&dptrs, sizeof(double*) * R, c->stream));
  std::vector<double*> hp(g->slot[par].begin(), g->slot[par].end());
  RCG_CUDA(c, cudaMemcpyAsync(dptrs, hp.data(), sizeof(double*) * R, cudaMemcpyHostToDevice, c->stream));
  sum_slots_kernel<<<(unsigned)std::min<size_t>((count + 255) / 256, 64), 256, 0, c->stream>>>(buf, dptrs, R, count);
  RCG_LAUNCH_CHECK(c);
  RCG_CUDA(c, cudaStreamSynchronize(c->stream));  // hp / dptrs lifetime (validation transport: simplicity first)
  cudaFreeAsync(dptrs, c->stream);
  RCG_CUDA(c, cudaEventRecord(g->consumed[par][me], c->stream));
  g->barrier();  // consumption events recorded before anyone reuses this parity
  return RCG_OK;
}

static int loop_halo(Ctx* c, const rcg_halo* H, double* dst_col) {
  LoopGroup* g = c->comm->loop;
  const int me = c->comm->rank, R = g->nranks;
  const int par = (int)(g->round[me] & 1);
  ++g->round[me];
  g->halo[me] = H;
  g->send_buf[me] = H->send_buf;
  RCG_CUDA(c, cudaEventRecord(g->ready[par][me], c->stream));   // after the pack kernel
  g->barrier();
  for (int q = 0; q < R; ++q) {
    if (q == me) continue;
    const rcg_halo* Hq = g->halo[q];
    const int64_t nr = H->recv_off[q + 1] - H->recv_off[q];
    if (nr <= 0) continue;
    RCG_CUDA(c, cudaStreamWaitEvent(c->stream, g->ready[par][q], 0));
    RCG_CUDA(c, cudaMemcpyAsync(dst_col + H->n_local + H->recv_off[q], g->send_buf[q] + Hq->send_off[me],
                                nr * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  }
  RCG_CUDA(c, cudaEventRecord(g->consumed[par][me], c->stream));
  g->barrier();
  return RCG_OK;
}

// RCG_COMM_FORCE=1: issue NCCL collectives even on one rank (exercises the
// NCCL calls, incl. their CUDA-graph capture, on a single GPU)
static bool comm_force() {   // read per call: tests switch it within one process
  const char* e = getenv("RCG_COMM_FORCE");
  return e && atoi(e) != 0;
}

bool comm_graphable(const Ctx* c) {
  const char* e = getenv("RCG_SHARDED_GRAPHS");
  return !(e && atoi(e) == 0) && c->comm && !c->comm->loop;
}

int allreduce_sum(Ctx* c, double* buf, size_t count) {
  if (!c->comm || count == 0) return RCG_OK;
  if (c->comm->nranks <= 1 && !(comm_force() && !c->comm->loop && c->comm->comm)) return RCG_OK;
  if (c->comm->loop) return loop_allreduce(c, buf, count);
  RCG_NCCL(c, c->comm->api.allReduce(buf, buf, count, kNcclFloat64, kNcclSum, c->comm->comm, c->stream));
  return RCG_OK;
}

__global__ void halo_pack_kernel(int64_t total, const int32_t* __restrict__ idx, ColSel src, const SolveState* st,
                                 double* __restrict__ out) {
  long long j = 0;
  if (st) j = st->j;  // when the solve already stopped this packs a stale column: harmless
  const double* s = src.at(j);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = s[idx[k]];
}

// Solve-loop variants: the column selector and the solve state are read from
// the device-resident argument block, not passed by value, so a captured batch
// graph stays valid when a later solve of the sequence has other history
// buffers or another state block (by value they were baked into the graph:
// the second system of a sharded sequence then read freed memory).
__global__ void halo_pack_kernel_ind(int64_t total, const int32_t* __restrict__ idx, const ColSel* __restrict__ srcp,
                                     const SolveState* const* __restrict__ stp, double* __restrict__ out) {
  const SolveState* st = *stp;
  const double* s = srcp->at(st->j);   // when the solve already stopped this packs a stale column: harmless
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = s[idx[k]];
}

__global__ void halo_unpack_kernel_ind(int64_t n_ghost, int64_t n_local, const double* __restrict__ in,
                                       const ColSel* __restrict__ dstp, const SolveState* const* __restrict__ stp) {
  const SolveState* st = *stp;
  double* d = dstp->at(st->j) + n_local;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_ghost; k += (int64_t)gridDim.x * blockDim.x)
    d[k] = in[k];
}

// The exchange runs with peers, or - RCG_COMM_FORCE=1 on a 1-rank NCCL
// communicator with a plan that lists ghost copies of the rank's own rows
// (two virtual slabs in one rank, tests/test_gpu_solver.py) - as a send /
// recv to self, so the whole pack -> ncclSend/ncclRecv -> unpack path and its
// CUDA-graph capture can be exercised on one GPU.
bool halo_active(const Ctx* c, const rcg_halo* H) {
  if (!H || !c->comm) return false;
  if (c->comm->nranks > 1) return true;
  return comm_force() && !c->comm->loop && c->comm->comm && H->n_ghost > 0;
}

static int halo_exchange_impl(Ctx* c, const rcg_halo* H, ColSel src, const SolveState* st, const ColSel* src_d,
                              const SolveState* const* st_d, double* dst_col);

int halo_exchange(Ctx* c, const rcg_halo* H, ColSel src, const SolveState* st, double* dst_col) {
  return halo_exchange_impl(c, H, src, st, nullptr, nullptr, dst_col);
}

// src_d / st_d non-null: the solve-loop form (arguments read from device memory)
static int halo_exchange_impl(Ctx* c, const rcg_halo* H, ColSel src, const SolveState* st, const ColSel* src_d,
                              const SolveState* const* st_d, double* dst_col) {
  if (!halo_active(c, H)) return RCG_OK;
  if (c->comm->loop) {
    // loopback: the single send buffer may be repacked only after every rank
    // consumed the previous exchange (events recorded before the last barrier)
    LoopGroup* g = c->comm->loop;
    for (int p = 0; p < 2; ++p)
      for (int q = 0; q < g->nranks; ++q) RCG_CUDA(c, cudaStreamWaitEvent(c->stream, g->consumed[p][q], 0));
  }
  const int64_t total = H->send_off[H->nranks];
  if (total > 0) {
    int64_t g = ceil_div(total, kThreads);
    if (g > 4 * c->num_sms) g = 4 * c->num_sms;
    if (src_d) halo_pack_kernel_ind<<<(unsigned)g, kThreads, 0, c->stream>>>(total, H->send_idx, src_d, st_d, H->send_buf);
    else halo_pack_kernel<<<(unsigned)g, kThreads, 0, c->stream>>>(total, H->send_idx, src, st, H->send_buf);
    RCG_LAUNCH_CHECK(c);
  }
  if (c->comm->loop) return loop_halo(c, H, dst_col);
  Nccl& api = c->comm->api;
  RCG_NCCL(c, api.groupStart());
  const bool self = c->comm->nranks <= 1;   // forced self exchange (halo_active)
  for (int q = 0; q < H->nranks; ++q) {
    if (q == H->rank && !self) continue;
    const int64_t ns = H->send_off[q + 1] - H->send_off[q];
    const int64_t nr = H->recv_off[q + 1] - H->recv_off[q];
    if (ns > 0) RCG_NCCL(c, api.send(H->send_buf + H->send_off[q], (size_t)ns, kNcclFloat64, q, c->comm->comm, c->stream));
    if (nr > 0)
      RCG_NCCL(c, api.recv(dst_col + H->n_local + H->recv_off[q], (size_t)nr, kNcclFloat64, q, c->comm->comm,
                           c->stream));
  }
  RCG_NCCL(c, api.groupEnd());
  return RCG_OK;
}

int halo_prepare(Ctx* c, const rcg_halo* H) {
  if (!H || H->n_ghost <= 0 || c->halo_recv_cap >= (size_t)H->n_ghost) return RCG_OK;
  RCG_CUDA(c, cudaStreamSynchronize(c->stream));   // the old buffer may still be read
  // captured batches hold the staging address in their recv / unpack nodes
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.second.exec);
  c->graphs.clear();
  if (c->halo_recv) cudaFree(c->halo_recv);
  c->halo_recv = nullptr;
  c->halo_recv_cap = 0;
  RCG_CUDA(c, cudaMalloc((void**)&c->halo_recv, sizeof(double) * (size_t)H->n_ghost));
  c->halo_recv_cap = (size_t)H->n_ghost;
  return RCG_OK;
}

int halo_exchange_dev(Ctx* c, const rcg_halo* H, const ColSel* src_d, const SolveState* const* st_d,
                      const ColSel* dst_d) {
  if (!halo_active(c, H)) return RCG_OK;
  if (H->n_ghost > (int64_t)c->halo_recv_cap)
    return set_error(c, RCG_ERR_CONTRACT, "halo staging not prepared (halo_prepare before the solve loop)");
  // received ghosts land at halo_recv + recv_off[q] (the exchange's "column"
  // is halo_recv - n_local), then move into the destination column at j
  int rc = halo_exchange_impl(c, H, ColSel{}, nullptr, src_d, st_d, c->halo_recv - H->n_local);
  if (rc) return rc;
  if (H->n_ghost > 0) {
    const int g = (int)std::min<int64_t>(ceil_div(H->n_ghost, (int64_t)kThreads), 2 * c->num_sms);
    halo_unpack_kernel_ind<<<g, kThreads, 0, c->stream>>>(H->n_ghost, H->n_local, c->halo_recv, dst_d, st_d);
    RCG_LAUNCH_CHECK(c);
  }
  return RCG_OK;
}

void comm_free(Ctx* c) {
  // captured batches hold this communicator's send / recv / allreduce nodes:
  // NCCL requires the graphs to go first (ncclCommDestroy otherwise blocks:
  // seen as a hang at process exit once halo send / recv were captured)
  cudaStreamSynchronize(c->stream);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.second.exec);
  c->graphs.clear();
  if (c->halo_recv) {
    cudaFree(c->halo_recv);
    c->halo_recv = nullptr;
    c->halo_recv_cap = 0;
  }
  if (c->comm) {
    if (!c->comm->loop && c->comm->comm && c->comm->api.commDestroy) c->comm->api.commDestroy(c->comm->comm);
    delete c->comm;
    c->comm = nullptr;
  }
}

}  // namespace rcg

using namespace rcg;

extern "C" int rcg_comm_unique_id(const char* nccl_lib, void* id_out) {
  if (!id_out) return RCG_ERR_CONTRACT;
  Nccl api;
  std::string err;
  int rc = load_nccl(nccl_lib, &api, &err);
  if (rc) return rc;
  ncclUniqueId id;
  if (api.getUniqueId(&id) != 0) return RCG_ERR_CUDA;
  std::memcpy(id_out, &id, sizeof(id));
  return RCG_OK;
}

extern "C" int rcg_comm_init(rcg_ctx* ctx, const char* nccl_lib, const void* id, int nranks, int rank) {
  if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return RCG_ERR_CONTRACT;
  comm_free(ctx);
  Comm* cm = new Comm();
  std::string err;
  int rc = load_nccl(nccl_lib, &cm->api, &err);
  if (rc) {
    delete cm;
    return set_error(ctx, rc, "%s", err.c_str());
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  cudaSetDevice(ctx->device);
  ncclResult_t r = cm->api.commInitRank(&cm->comm, nranks, uid, rank);
  if (r != 0) {
    const char* s = cm->api.errStr(r);
    delete cm;
    return set_error(ctx, RCG_ERR_CUDA, "ncclCommInitRank: %s", s);
  }
  cm->nranks = nranks;
  cm->rank = rank;
  ctx->comm = cm;
  return RCG_OK;
}

extern "C" int rcg_comm_destroy(rcg_ctx* ctx) {
  if (!ctx) return RCG_ERR_CONTRACT;
  cudaStreamSynchronize(ctx->stream);
  comm_free(ctx);
  return RCG_OK;
}

extern "C" int rcg_allreduce_sum(rcg_ctx* ctx, double* buf, int64_t count) {
  if (!ctx) return RCG_ERR_CONTRACT;
  return allreduce_sum(ctx, buf, (size_t)count);
}

extern "C" int rcg_halo_exchange(rcg_ctx* ctx, const rcg_halo* H, double* vec) {
  if (!ctx || !H) return RCG_ERR_CONTRACT;
  return halo_exchange(ctx, H, colsel(vec), nullptr, vec);
}

extern "C" int rcg_loop_group_create(int nranks, void** out) {
  if (!out || nranks < 1 || nranks > 64) return RCG_ERR_CONTRACT;
  LoopGroup* g = new LoopGroup();
  g->nranks = nranks;
  for (int p = 0; p < 2; ++p) {
    g->slot[p].assign(nranks, nullptr);
    g->slot_cap[p].assign(nranks, 0);
    g->ready[p].resize(nranks);
    g->consumed[p].resize(nranks);
    for (int r = 0; r < nranks; ++r) {
      cudaEventCreateWithFlags(&g->ready[p][r], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&g->consumed[p][r], cudaEventDisableTiming);
      cudaEventRecord(g->consumed[p][r], 0);  // "consumed" initially
    }
  }
  g->halo.assign(nranks, nullptr);
  g->send_buf.assign(nranks, nullptr);
  cudaDeviceSynchronize();
  *out = g;
  return RCG_OK;
}

extern "C" void rcg_loop_group_destroy(void* gp) {
  LoopGroup* g = (LoopGroup*)gp;
  if (!g) return;
  cudaDeviceSynchronize();
  for (int p = 0; p < 2; ++p)
    for (int r = 0; r < g->nranks; ++r) {
      if (g->slot[p][r]) cudaFree(g->slot[p][r]);
      cudaEventDestroy(g->ready[p][r]);
      cudaEventDestroy(g->consumed[p][r]);
    }
  delete g;
}

extern "C" int rcg_comm_init_loopback(rcg_ctx* ctx, void* group, int rank) {
  LoopGroup* g = (LoopGroup*)group;
  if (!ctx || !g || rank < 0 || rank >= g->nranks) return RCG_ERR_CONTRACT;
  comm_free(ctx);
  Comm* cm = new Comm();
  cm->nranks = g->nranks;
  cm->rank = rank;
  cm->loop = g;
  ctx->comm = cm;
  return RCG_OK;
}
