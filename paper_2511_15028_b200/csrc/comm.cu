// Multi-GPU plumbing of the C ABI ("queries may run concurrently on a shared immutable
// tree", :645 "reports are merged deterministically by query index"): the packed device image of a tree is
// replicated with ONE ncclBroadcast, the query index space is cut into contiguous ranges (scion_partition), and
// result records are gathered by query index.  There is no collective inside a traversal launch.
//
// NCCL is bound at RUN time (dlopen of libnccl.so.2): the library has no link-time NCCL dependency, a process that
// already carries an NCCL (torch's bundled one) gets that very instance — so a caller's ncclComm_t can be adopted —
// and single-GPU users need no NCCL at all.  Only the stable core API is used (GetUniqueId, CommInitRank,
// CommInitAll, Broadcast, AllGather, Group*, CommDestroy).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "host/dtree.hpp"
#include "scion_b200.h"

static_assert(SCION_NCCL_UNIQUE_ID_BYTES == sizeof(ncclUniqueId), "scion_b200.h must carry NCCL's unique-id size");

struct scion_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
  bool owns = true;
};

namespace {

using scion::abi_fail;

struct Nccl {
  void* handle = nullptr;
  std::string why;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommCuDevice)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {getenv("SCION_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm || !*nm) continue;
      n.handle = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.handle) break;
      n.why = dlerror();
    }
    if (!n.handle) return;
    bool ok = true;
    auto sym = [&](const char* name, auto& fp) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(n.handle, name));
      if (!fp) { ok = false; n.why = std::string("libnccl lacks ") + name; }
    };
    sym("ncclGetVersion", n.GetVersion);
    sym("ncclGetUniqueId", n.GetUniqueId);
    sym("ncclCommInitRank", n.CommInitRank);
    sym("ncclCommInitAll", n.CommInitAll);
    sym("ncclCommDestroy", n.CommDestroy);
    sym("ncclCommCount", n.CommCount);
    sym("ncclCommUserRank", n.CommUserRank);
    sym("ncclCommCuDevice", n.CommCuDevice);
    sym("ncclBroadcast", n.Broadcast);
    sym("ncclAllGather", n.AllGather);
    sym("ncclGroupStart", n.GroupStart);
    sym("ncclGroupEnd", n.GroupEnd);
    sym("ncclGetErrorString", n.GetErrorString);
    if (!ok) { dlclose(n.handle); n.handle = nullptr; }
  });
  return n.handle ? &n : nullptr;
}

#define NEED_NCCL()                                                                                                \
  const Nccl* N = nccl();                                                                                          \
  if (!N) return abi_fail(SCION_ERR_ARG, "NCCL is not available in this process (dlopen libnccl.so.2 failed; set SCION_NCCL_LIB)")
#define NCCL_OK(expr)                                                                                              \
  do {                                                                                                             \
    ncclResult_t r__ = (expr);                                                                                     \
    if (r__ != ncclSuccess) return abi_fail(SCION_ERR_CUDA, std::string(#expr) + ": " + N->GetErrorString(r__));   \
  } while (0)
#define CU_OK(expr)                                                                                                \
  do {                                                                                                             \
    cudaError_t e__ = (expr);                                                                                      \
    if (e__ != cudaSuccess) return abi_fail(e__ == cudaErrorNoDevice ? SCION_ERR_NO_DEVICE : SCION_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__)); \
  } while (0)

// receiving side of a broadcast: adopt a freshly allocated image
int tree_from_received(uint8_t* image, uint64_t bytes, int device, scion_dtree** out) {
  int rc = scion_dtree_from_image(nullptr, image, bytes, device, /*adopt=*/1, out);
  if (rc) cudaFree(image);
  return rc;
}

}  // namespace

extern "C" {

int scion_nccl_version(int* out) {
  NEED_NCCL();
  int v = 0;
  NCCL_OK(N->GetVersion(&v));
  if (out) *out = v;
  return SCION_OK;
}

int scion_comm_unique_id(uint8_t id[SCION_NCCL_UNIQUE_ID_BYTES]) {
  if (!id) return abi_fail(SCION_ERR_ARG, "null id");
  NEED_NCCL();
  ncclUniqueId u;
  NCCL_OK(N->GetUniqueId(&u));
  memcpy(id, &u, sizeof(u));
  return SCION_OK;
}

int scion_comm_init_rank(const uint8_t id[SCION_NCCL_UNIQUE_ID_BYTES], int nranks, int rank, int device, scion_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return abi_fail(SCION_ERR_ARG, "bad communicator arguments");
  NEED_NCCL();
  CU_OK(cudaSetDevice(device));
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  auto* c = new scion_comm();
  c->rank = rank; c->nranks = nranks; c->device = device;
  ncclResult_t r = N->CommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) { delete c; return abi_fail(SCION_ERR_CUDA, std::string("ncclCommInitRank: ") + N->GetErrorString(r)); }
  *out = c;
  return SCION_OK;
}

int scion_comm_init_all(int ndev, const int* devices, scion_comm** out) {
  if (ndev < 1 || !out) return abi_fail(SCION_ERR_ARG, "bad communicator arguments");
  NEED_NCCL();
  int have = 0;
  CU_OK(cudaGetDeviceCount(&have));
  std::vector<int> devs((size_t)ndev);
  for (int i = 0; i < ndev; i++) {
    devs[(size_t)i] = devices ? devices[i] : i;
    if (devs[(size_t)i] < 0 || devs[(size_t)i] >= have) return abi_fail(SCION_ERR_ARG, "scion_comm_init_all: device " + std::to_string(devs[(size_t)i]) + " of " + std::to_string(have) + " does not exist");
  }
  std::vector<ncclComm_t> comms((size_t)ndev);
  NCCL_OK(N->CommInitAll(comms.data(), ndev, devs.data()));
  for (int i = 0; i < ndev; i++) {
    auto* c = new scion_comm();
    c->comm = comms[(size_t)i]; c->rank = i; c->nranks = ndev; c->device = devs[(size_t)i];
    out[i] = c;
  }
  return SCION_OK;
}

int scion_comm_adopt(void* nccl_comm, scion_comm** out) {
  if (!nccl_comm || !out) return abi_fail(SCION_ERR_ARG, "null communicator");
  NEED_NCCL();
  auto* c = new scion_comm();
  c->comm = (ncclComm_t)nccl_comm;
  c->owns = false;
  ncclResult_t r = N->CommCount(c->comm, &c->nranks);
  if (r == ncclSuccess) r = N->CommUserRank(c->comm, &c->rank);
  if (r == ncclSuccess) r = N->CommCuDevice(c->comm, &c->device);
  if (r != ncclSuccess) { delete c; return abi_fail(SCION_ERR_CUDA, std::string("scion_comm_adopt: ") + N->GetErrorString(r)); }
  *out = c;
  return SCION_OK;
}

int scion_comm_rank(const scion_comm* c) { return c ? c->rank : -1; }
int scion_comm_size(const scion_comm* c) { return c ? c->nranks : 0; }
int scion_comm_device(const scion_comm* c) { return c ? c->device : -1; }
void scion_comm_free(scion_comm* c) {
  if (!c) return;
  const Nccl* N = nccl();
  if (c->owns && c->comm && N) { cudaSetDevice(c->device); N->CommDestroy(c->comm); }
  delete c;
}

// One process per GPU.  The root passes its resident tree, every other rank passes NULL; all ranks return with a
// tree on their communicator's device (the root gets its own tree back).  Two collectives: the 1 KB image header
// (it carries the size), then the whole packed image.
int scion_dtree_broadcast(scion_dtree* root_tree, int root, scion_comm* comm, void* stream, scion_dtree** out) {
  if (!comm || !out || root < 0 || root >= comm->nranks) return abi_fail(SCION_ERR_ARG, "bad broadcast arguments");
  const bool is_root = comm->rank == root;
  if (is_root != (root_tree != nullptr)) return abi_fail(SCION_ERR_ARG, "scion_dtree_broadcast: exactly the root rank passes a tree");
  if (is_root && root_tree->device != comm->device) return abi_fail(SCION_ERR_ARG, "the root's tree lives on another device than its communicator");
  NEED_NCCL();
  cudaStream_t s = (cudaStream_t)stream;
  CU_OK(cudaSetDevice(comm->device));
  uint8_t* hdr = nullptr;
  if (is_root) hdr = root_tree->image;
  else CU_OK(cudaMalloc(&hdr, scion::kHeaderBytes));
  ncclResult_t r = N->Broadcast(hdr, hdr, scion::kHeaderBytes, ncclUint8, root, comm->comm, s);
  if (r != ncclSuccess) { if (!is_root) cudaFree(hdr); return abi_fail(SCION_ERR_CUDA, std::string("ncclBroadcast(header): ") + N->GetErrorString(r)); }
  uint64_t total = 0;
  if (is_root) {
    total = root_tree->header.total_bytes;
  } else {
    scion::ImageHeader h;
    cudaError_t e = cudaMemcpyAsync(&h, hdr, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(hdr);
    CU_OK(e);
    if (h.magic != scion::kImageMagic || h.total_bytes < scion::kHeaderBytes) return abi_fail(SCION_ERR_ARG, "scion_dtree_broadcast: received a corrupt image header");
    total = h.total_bytes;
  }
  uint8_t* image = is_root ? root_tree->image : nullptr;
  if (!is_root) CU_OK(cudaMalloc(&image, total));
  r = N->Broadcast(image, image, total, ncclUint8, root, comm->comm, s);
  if (r != ncclSuccess) { if (!is_root) cudaFree(image); return abi_fail(SCION_ERR_CUDA, std::string("ncclBroadcast(image): ") + N->GetErrorString(r)); }
  if (is_root) { *out = root_tree; return SCION_OK; }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) { cudaFree(image); CU_OK(e); }
  return tree_from_received(image, total, comm->device, out);
}

// Single process, one communicator per device (scion_comm_init_all): trees[root] is resident, every other entry is
// filled in.  streams may be NULL (default stream of each device).
int scion_dtree_broadcast_all(scion_dtree* root_tree, int root, scion_comm* const* comms, int n, void* const* streams, scion_dtree** out) {
  if (!root_tree || !comms || !out || n < 1 || root < 0 || root >= n) return abi_fail(SCION_ERR_ARG, "bad broadcast arguments");
  NEED_NCCL();
  for (int i = 0; i < n; i++)
    if (!comms[i] || comms[i]->nranks != n || comms[i]->rank != i) return abi_fail(SCION_ERR_ARG, "scion_dtree_broadcast_all: comms must be the array scion_comm_init_all returned");
  if (root_tree->device != comms[root]->device) return abi_fail(SCION_ERR_ARG, "the root's tree lives on another device than its communicator");
  const uint64_t total = root_tree->header.total_bytes;  // one process: the size needs no collective
  std::vector<uint8_t*> img((size_t)n, nullptr);
  auto cleanup = [&] { for (int i = 0; i < n; i++) if (i != root && img[(size_t)i]) { cudaSetDevice(comms[i]->device); cudaFree(img[(size_t)i]); } };
  for (int i = 0; i < n; i++) {
    if (i == root) { img[(size_t)i] = root_tree->image; continue; }
    cudaError_t e = cudaSetDevice(comms[i]->device);
    if (e == cudaSuccess) e = cudaMalloc(&img[(size_t)i], total);
    if (e != cudaSuccess) { cleanup(); CU_OK(e); }
  }
  ncclResult_t r = N->GroupStart();
  for (int i = 0; i < n && r == ncclSuccess; i++) {
    cudaSetDevice(comms[i]->device);
    r = N->Broadcast(img[(size_t)i], img[(size_t)i], total, ncclUint8, root, comms[i]->comm, streams ? (cudaStream_t)streams[i] : nullptr);
  }
  ncclResult_t r2 = N->GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) { cleanup(); return abi_fail(SCION_ERR_CUDA, std::string("ncclBroadcast(image): ") + N->GetErrorString(r)); }
  for (int i = 0; i < n; i++) {
    cudaSetDevice(comms[i]->device);
    cudaError_t e = cudaStreamSynchronize(streams ? (cudaStream_t)streams[i] : nullptr);
    if (e != cudaSuccess) { cleanup(); CU_OK(e); }
  }
  for (int i = 0; i < n; i++) {
    if (i == root) { out[i] = root_tree; continue; }
    int rc = tree_from_received(img[(size_t)i], total, comms[i]->device, &out[i]);
    img[(size_t)i] = nullptr;
    if (rc) { for (int k = 0; k < i; k++) if (k != root) { scion_dtree_free(out[k]); out[k] = nullptr; } cleanup(); return rc; }
  }
  return SCION_OK;
}

// Gather of result records by query index: rank r holds the records of scion_partition(n_total, r, nranks) in
// d_part; every rank receives all n_total records, in query order, in d_full (which may contain d_part at its own
// offset: in place).  Equal shares use ncclAllGather, ragged ones one grouped ncclBroadcast per rank.
int scion_gather_results(scion_comm* comm, const void* d_part, uint64_t n_total, uint32_t record_bytes, void* d_full, void* stream) {
  if (!comm || !d_full || (!d_part && n_total) || record_bytes == 0) return abi_fail(SCION_ERR_ARG, "bad gather arguments");
  NEED_NCCL();
  cudaStream_t s = (cudaStream_t)stream;
  CU_OK(cudaSetDevice(comm->device));
  const int R = comm->nranks;
  uint64_t first = 0, count = 0;
  scion_partition(n_total, comm->rank, R, &first, &count);
  uint8_t* full = (uint8_t*)d_full;
  if (n_total == 0) return SCION_OK;
  (void)first;
  if (n_total % (uint64_t)R == 0) {  // a one-rank communicator goes through NCCL too (copy, or nothing when in place)
    NCCL_OK(N->AllGather(d_part, d_full, count * record_bytes, ncclUint8, comm->comm, s));
    return SCION_OK;
  }
  ncclResult_t r = N->GroupStart();
  for (int k = 0; k < R && r == ncclSuccess; k++) {
    uint64_t f = 0, c = 0;
    scion_partition(n_total, k, R, &f, &c);
    uint8_t* dst = full + f * record_bytes;
    r = N->Broadcast(k == comm->rank ? d_part : (const void*)dst, dst, c * record_bytes, ncclUint8, k, comm->comm, s);
  }
  ncclResult_t r2 = N->GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return abi_fail(SCION_ERR_CUDA, std::string("scion_gather_results: ") + N->GetErrorString(r));
  return SCION_OK;
}

// single-process form: d_parts[i] on device i -> d_fulls[i] (all records) on device i
int scion_gather_results_all(scion_comm* const* comms, int n, const void* const* d_parts, uint64_t n_total, uint32_t record_bytes, void* const* d_fulls,
                             void* const* streams) {
  if (!comms || !d_parts || !d_fulls || n < 1 || record_bytes == 0) return abi_fail(SCION_ERR_ARG, "bad gather arguments");
  NEED_NCCL();
  if (n_total == 0) return SCION_OK;
  ncclResult_t r = N->GroupStart();
  for (int i = 0; i < n && r == ncclSuccess; i++) {
    cudaSetDevice(comms[i]->device);
    cudaStream_t s = streams ? (cudaStream_t)streams[i] : nullptr;
    for (int k = 0; k < n && r == ncclSuccess; k++) {
      uint64_t f = 0, c = 0;
      scion_partition(n_total, k, n, &f, &c);
      uint8_t* dst = (uint8_t*)d_fulls[i] + f * record_bytes;
      r = N->Broadcast(k == i ? d_parts[i] : (const void*)dst, dst, c * record_bytes, ncclUint8, k, comms[i]->comm, s);
    }
  }
  ncclResult_t r2 = N->GroupEnd();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return abi_fail(SCION_ERR_CUDA, std::string("scion_gather_results_all: ") + N->GetErrorString(r));
  return SCION_OK;
}

}  // extern "C"
