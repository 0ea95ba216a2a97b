// comm.cu — NCCL for the column-sharded dense mode (BASELINE config 3
// "column-sharded runs"): rank r owns the columns [d_offset, d_offset + D_r) of Phi and
// the matching rows of every D-vector; each CG iteration sums W = Phi P over ranks and the
// per-column dot products (gamma_j, rho_j -- or, single-reduction CG, gamma_j, delta1_j, delta2_j in
// one all-reduce, reading R23) before the step lengths are taken.
//
// NCCL is resolved at run time (dlopen of the libnccl.so.2 already mapped into the process —
// torch's — or the system one), so the library has no link-time NCCL dependency and a
// single-GPU user never loads it.  Collectives are enqueued on the context stream (no host
// synchronisation), so the sharded E-step is still captured into one CUDA graph.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <string>

#include "internal.cuh"

namespace cofem {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl(std::string& err) {
  static NcclApi api;
  static bool tried = false;
  if (tried) { if (!api.ok) err = "NCCL not available"; return api; }
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);   // torch's, if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { err = std::string("dlopen libnccl.so.2: ") + dlerror(); return api; }
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.CommAbort = (decltype(api.CommAbort))dlsym(h, "ncclCommAbort");
  api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
  api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
  api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GetErrorString && api.Send &&
           api.Recv && api.GroupStart && api.GroupEnd && api.Broadcast;
  if (!api.ok) err = "libnccl.so.2 lacks required symbols";
  return api;
}

cofem_status comm_init(Ctx* c, int rank, int world, const uint8_t* id) {
  NcclApi& a = nccl(c->err);
  if (!a.ok) return COFEM_ERR_NCCL;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ncclComm_t comm;
  ncclResult_t r = a.CommInitRank(&comm, world, uid, rank);
  if (r != ncclSuccess) { c->err = std::string("ncclCommInitRank: ") + a.GetErrorString(r); return COFEM_ERR_NCCL; }
  c->comm = comm;
  return COFEM_OK;
}

void comm_destroy(Ctx* c) {
  if (!c->comm) return;
  std::string e;
  NcclApi& a = nccl(e);
  // ncclCommAbort does not wait on peers (a rank being torn down must not block on the
  // others' progress, e.g. at interpreter exit); fall back to ncclCommDestroy
  if (a.ok) (a.CommAbort ? a.CommAbort : a.CommDestroy)((ncclComm_t)c->comm);
  c->comm = nullptr;
}

// In-place sum over ranks on the context stream; dtype 0 = fp32, 1 = fp64.
cofem_status comm_allreduce(Ctx* c, void* buf, size_t count, int dtype) {
  NcclApi& a = nccl(c->err);
  if (!a.ok || !c->comm) return COFEM_ERR_NCCL;
  ncclResult_t r = a.AllReduce(buf, buf, count, dtype ? ncclFloat64 : ncclFloat32, ncclSum, (ncclComm_t)c->comm,
                               c->stream);
  if (c->comm_depth == 0) c->collectives++;
  if (r != ncclSuccess) { c->err = std::string("ncclAllReduce: ") + a.GetErrorString(r); return COFEM_ERR_NCCL; }
  return COFEM_OK;
}

cofem_status comm_group(Ctx* c, bool begin) {
  NcclApi& a = nccl(c->err);
  if (!a.ok || !c->comm) return COFEM_ERR_NCCL;
  ncclResult_t r = begin ? a.GroupStart() : a.GroupEnd();
  c->comm_depth += begin ? 1 : -1;
  if (!begin && c->comm_depth == 0) c->collectives++;
  if (r != ncclSuccess) { c->err = std::string("ncclGroup: ") + a.GetErrorString(r); return COFEM_ERR_NCCL; }
  return COFEM_OK;
}

// In-place broadcast from `root` on the context stream (probe-parallel: mu = x0 from rank 0).
cofem_status comm_bcast(Ctx* c, void* buf, size_t count, int dtype, int root) {
  NcclApi& a = nccl(c->err);
  if (!a.ok || !c->comm) return COFEM_ERR_NCCL;
  ncclResult_t r = a.Broadcast(buf, buf, count, dtype ? ncclFloat64 : ncclFloat32, root, (ncclComm_t)c->comm, c->stream);
  if (c->comm_depth == 0) c->collectives++;
  if (r != ncclSuccess) { c->err = std::string("ncclBroadcast: ") + a.GetErrorString(r); return COFEM_ERR_NCCL; }
  return COFEM_OK;
}

// Ring halo exchange (D-sharded convolution): this rank's first block goes to the left
// neighbour (it is that rank's right halo), its last block to the right neighbour; the
// matching blocks arrive in recv_left / recv_right.  count elements of dtype per side.
cofem_status comm_halo(Ctx* c, const void* send_left, const void* send_right, void* recv_left, void* recv_right,
                       size_t count, int dtype) {
  NcclApi& a = nccl(c->err);
  if (!a.ok || !c->comm) return COFEM_ERR_NCCL;
  const int left = (c->rank + c->world - 1) % c->world, right = (c->rank + 1) % c->world;
  const ncclDataType_t t = dtype ? ncclFloat64 : ncclFloat32;
  ncclComm_t cm = (ncclComm_t)c->comm;
  ncclResult_t r = a.GroupStart();
  if (r == ncclSuccess) r = a.Send(send_left, count, t, left, cm, c->stream);
  if (r == ncclSuccess) r = a.Recv(recv_right, count, t, right, cm, c->stream);
  if (r == ncclSuccess) r = a.Send(send_right, count, t, right, cm, c->stream);
  if (r == ncclSuccess) r = a.Recv(recv_left, count, t, left, cm, c->stream);
  ncclResult_t r2 = a.GroupEnd();
  if (c->comm_depth == 0) c->collectives++;
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) { c->err = std::string("NCCL halo exchange: ") + a.GetErrorString(r); return COFEM_ERR_NCCL; }
  return COFEM_OK;
}

}  // namespace cofem

extern "C" cofem_status cofem_get_unique_id(uint8_t id[128]) {
  std::string err;
  cofem::NcclApi& a = cofem::nccl(err);
  if (!a.ok || !id) return COFEM_ERR_NCCL;
  ncclUniqueId uid;
  if (a.GetUniqueId(&uid) != ncclSuccess) return COFEM_ERR_NCCL;
  memcpy(id, &uid, sizeof uid);
  return COFEM_OK;
}
