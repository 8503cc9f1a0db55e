// Communicator of the slab decomposition (dist.h).
#include "dist.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "engine.h"

namespace hadr {

// ---------------------------------------------------------------------------
// NCCL, opened at run time (no link-time dependency of libhadr on NCCL)
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi a;
  if (a.h) return a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw std::runtime_error("NCCL not found (libnccl.so.2)");
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + n);
    return p;
  };
  a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
  a.Send = (decltype(a.Send))sym("ncclSend");
  a.Recv = (decltype(a.Recv))sym("ncclRecv");
  a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
  a.Broadcast = (decltype(a.Broadcast))sym("ncclBroadcast");
  a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
  a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
  a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
  a.h = h;
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL error in ") + what + ": " + nccl_api().GetErrorString(r));
}

void host_check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string("host communicator callback failed: ") + what);
}

Comm* g_comm = nullptr;

void red_gather(void* ctx, cudaStream_t s) {
  Comm* c = (Comm*)ctx;
  c->allgather(c->red.buf, c->red.all, 4 * sizeof(double), s);
}
}  // namespace

char* Comm::stage(size_t bytes) {
  if (bytes > hstage_bytes) {
    if (hstage) cudaFreeHost(hstage);
    HADR_CUDA(cudaMallocHost(&hstage, bytes));
    hstage_bytes = bytes;
  }
  return (char*)hstage;
}

void Comm::group_start() {
  if (kind == 1) nccl_check(nccl_api().GroupStart(), "ncclGroupStart");
}
void Comm::group_end() {
  if (kind == 1) nccl_check(nccl_api().GroupEnd(), "ncclGroupEnd");
}

void Comm::allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s) {
  if (kind == 1) {
    nccl_check(nccl_api().AllGather(dsend, drecv, bytes, ncclUint8, (ncclComm_t)nccl, s), "ncclAllGather");
    return;
  }
  char* h = stage(bytes * (size + 1));
  HADR_CUDA(cudaMemcpyAsync(h, dsend, bytes, cudaMemcpyDeviceToHost, s));
  HADR_CUDA(cudaStreamSynchronize(s));
  host_check(h_allgather(h, h + bytes, (long long)bytes), "allgather");
  HADR_CUDA(cudaMemcpyAsync(drecv, h + bytes, bytes * size, cudaMemcpyHostToDevice, s));
  HADR_CUDA(cudaStreamSynchronize(s));
}

void Comm::bcast(void* dbuf, size_t bytes, int root, cudaStream_t s) {
  if (bytes == 0) return;
  if (kind == 1) {
    nccl_check(nccl_api().Broadcast(dbuf, dbuf, bytes, ncclUint8, root, (ncclComm_t)nccl, s), "ncclBroadcast");
    return;
  }
  char* h = stage(bytes);
  if (rank == root) {
    HADR_CUDA(cudaMemcpyAsync(h, dbuf, bytes, cudaMemcpyDeviceToHost, s));
    HADR_CUDA(cudaStreamSynchronize(s));
  }
  host_check(h_bcast(h, (long long)bytes, root), "bcast");
  if (rank != root) {
    HADR_CUDA(cudaMemcpyAsync(dbuf, h, bytes, cudaMemcpyHostToDevice, s));
    HADR_CUDA(cudaStreamSynchronize(s));
  }
}

void Comm::halo(void* v, size_t plane_bytes, int nown, int h, cudaStream_t s) {
  if (size == 1) return;
  char* p = (char*)v;
  const size_t hb = plane_bytes * h;
  const int lo = rank > 0 ? rank - 1 : -1, hi = rank < size - 1 ? rank + 1 : -1;
  char* first = p;                                 // owned planes [0, h)
  char* last = p + plane_bytes * (nown - h);       // owned planes [nown - h, nown)
  char* below = p - hb;                            // halo planes [-h, 0)
  char* above = p + plane_bytes * nown;            // halo planes [nown, nown + h)
  if (kind == 1) {
    auto& a = nccl_api();
    ncclComm_t c = (ncclComm_t)nccl;
    nccl_check(a.GroupStart(), "ncclGroupStart");
    if (lo >= 0) {
      nccl_check(a.Send(first, hb, ncclUint8, lo, c, s), "ncclSend");
      nccl_check(a.Recv(below, hb, ncclUint8, lo, c, s), "ncclRecv");
    }
    if (hi >= 0) {
      nccl_check(a.Send(last, hb, ncclUint8, hi, c, s), "ncclSend");
      nccl_check(a.Recv(above, hb, ncclUint8, hi, c, s), "ncclRecv");
    }
    nccl_check(a.GroupEnd(), "ncclGroupEnd");
    return;
  }
  char* hs = stage(4 * hb);
  HADR_CUDA(cudaMemcpyAsync(hs, first, hb, cudaMemcpyDeviceToHost, s));
  HADR_CUDA(cudaMemcpyAsync(hs + hb, last, hb, cudaMemcpyDeviceToHost, s));
  HADR_CUDA(cudaStreamSynchronize(s));
  // phase 1: first planes down, upper halo from above; phase 2: last planes up, lower halo from below
  host_check(h_sendrecv(hs, lo >= 0 ? (long long)hb : 0, lo, hs + 2 * hb, hi >= 0 ? (long long)hb : 0, hi),
             "sendrecv");
  host_check(h_sendrecv(hs + hb, hi >= 0 ? (long long)hb : 0, hi, hs + 3 * hb, lo >= 0 ? (long long)hb : 0, lo),
             "sendrecv");
  if (hi >= 0) HADR_CUDA(cudaMemcpyAsync(above, hs + 2 * hb, hb, cudaMemcpyHostToDevice, s));
  if (lo >= 0) HADR_CUDA(cudaMemcpyAsync(below, hs + 3 * hb, hb, cudaMemcpyHostToDevice, s));
  HADR_CUDA(cudaStreamSynchronize(s));
}

void Comm::allreduce_or_u64(unsigned long long* v, int n, cudaStream_t s) {
  if (size == 1) return;
  const size_t bytes = n * sizeof(unsigned long long);
  if (!dscratch) dscratch = dalloc<unsigned long long>(64 * 16);
  if ((size_t)size * bytes > 64 * 16 * sizeof(unsigned long long)) throw std::runtime_error("allreduce_or: too large");
  unsigned long long* d = (unsigned long long*)dscratch;
  std::vector<unsigned long long> all((size_t)size * n);
  HADR_CUDA(cudaMemcpyAsync(d, v, bytes, cudaMemcpyHostToDevice, s));
  allgather(d, d + n, bytes, s);
  HADR_CUDA(cudaMemcpyAsync(all.data(), d + n, bytes * size, cudaMemcpyDeviceToHost, s));
  HADR_CUDA(cudaStreamSynchronize(s));
  for (int r = 0; r < size; ++r)
    for (int q = 0; q < n; ++q) v[q] |= all[(size_t)r * n + q];
}

Comm* dist_comm() { return g_comm; }
int g_dist_min_planes = 16;
int g_dist_levels = 0;
double g_dist_min_work = 8e6;

static void install(Comm* c) {
  c->red.size = c->size;
  c->red.buf = dalloc<double>(4);
  c->red.all = dalloc<double>(4 * c->size);
  HADR_CUDA(cudaMemset(c->red.buf, 0, 4 * sizeof(double)));
  c->red.gather = red_gather;
  c->red.ctx = c;
  dist_finalize();
  g_comm = c;
}

int dist_nccl_unique_id(char* out) {
  ncclUniqueId id;
  nccl_check(nccl_api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int dist_init_nccl(int rank, int size, const char* unique_id) {
  if (size < 1 || rank < 0 || rank >= size) throw ValueError("bad rank / size");
  Ctx::get();
  ncclUniqueId id;
  std::memcpy(id.internal, unique_id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t nc;
  nccl_check(nccl_api().CommInitRank(&nc, size, id, rank), "ncclCommInitRank");
  Comm* c = new Comm();
  c->rank = rank;
  c->size = size;
  c->kind = 1;
  c->nccl = nc;
  install(c);
  return 0;
}

int dist_init_host(int rank, int size, HostAllgather ag, HostSendrecv sr, HostBcast bc) {
  if (size < 1 || rank < 0 || rank >= size) throw ValueError("bad rank / size");
  if (!ag || !sr || !bc) throw ValueError("host communicator needs allgather, sendrecv and bcast callbacks");
  Ctx::get();
  Comm* c = new Comm();
  c->rank = rank;
  c->size = size;
  c->kind = 2;
  c->h_allgather = ag;
  c->h_sendrecv = sr;
  c->h_bcast = bc;
  install(c);
  return 0;
}

void dist_finalize() {
  Comm* c = g_comm;
  g_comm = nullptr;
  if (!c) return;
  cudaStreamSynchronize(Ctx::get().stream);
  if (c->kind == 1 && c->nccl) nccl_api().CommDestroy((ncclComm_t)c->nccl);
  dfree(c->red.buf);
  dfree(c->red.all);
  // host staging / scratch intentionally kept small; released with the process
  delete c;
}

std::vector<int> slab_bounds(int n1, int size, int align) {
  std::vector<int> b(size + 1, 0);
  b[size] = n1;
  const int cells = n1 - 1;
  for (int r = 1; r < size; ++r) {
    const long t = (long)cells * r / size;
    int v = (int)((t + align / 2) / align) * align;
    b[r] = v;
  }
  for (int r = 1; r <= size; ++r)
    if (b[r] - b[r - 1] < 1) return {};
  return b;
}

}  // namespace hadr
