// Row-sharded multi-GPU plumbing: NCCL (loaded with dlopen, so librcg.so
// has no hard NCCL dependency) for the halo exchange of SpMV ghost entries
// and the packed fp64 allreduces of the per-iteration reduction slots
// (SURVEY.md §8(e)).  One process per GPU; every rank holds a contiguous row
// slab, and the ghost values it reads live in a region appended after its
// n_local entries of every SpMV-input column (W[:, j], C[:, c], x0).
#include "rcg_internal.cuh"
#include "comm.cuh"

#include <dlfcn.h>
#include <cstring>

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

struct Comm {
  Nccl api;
  ncclComm_t comm = nullptr;
  int nranks = 1;
  int rank = 0;
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

int allreduce_sum(Ctx* c, double* buf, size_t count) {
  if (!c->comm || c->comm->nranks <= 1 || count == 0) return RCG_OK;
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

int halo_exchange(Ctx* c, const rcg_halo* H, ColSel src, const SolveState* st, double* dst_col) {
  if (!H || !c->comm || c->comm->nranks <= 1) return RCG_OK;
  const int64_t total = H->send_off[H->nranks];
  if (total > 0) {
    int64_t g = ceil_div(total, kThreads);
    if (g > 4 * c->num_sms) g = 4 * c->num_sms;
    halo_pack_kernel<<<(unsigned)g, kThreads, 0, c->stream>>>(total, H->send_idx, src, st, H->send_buf);
    RCG_LAUNCH_CHECK(c);
  }
  Nccl& api = c->comm->api;
  RCG_NCCL(c, api.groupStart());
  for (int q = 0; q < H->nranks; ++q) {
    if (q == H->rank) continue;
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

void comm_free(Ctx* c) {
  if (c->comm) {
    if (c->comm->comm && c->comm->api.commDestroy) c->comm->api.commDestroy(c->comm->comm);
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
