// Multi-GPU slab decomposition: one process per GPU, axis-0
// slabs of the fine grid and of every distributed coarse level, coarse levels
// below a plane threshold agglomerated (replicated on every rank).
//
// Communicator backends:
//   NCCL (kind 1)  — one GPU per rank; libnccl.so.2 is opened at run time (the
//                    copy torch already loaded, else the system one).  Halo
//                    exchange = grouped ncclSend/ncclRecv of contiguous planes,
//                    reductions = ncclAllGather of 4 doubles, agglomeration =
//                    grouped ncclBroadcast; all stream-ordered and capturable
//                    in the K-cycle CUDA graph.
//   host (kind 2)  — blocking host callbacks (e.g. torch.distributed gloo):
//                    several ranks may share one GPU because no kernel ever
//                    waits on another rank; the stream is synchronised around
//                    every exchange and nothing is graph-captured.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "kernels.cuh"

namespace hadr {

constexpr int kHalo = 2;  // vector halo planes: the largest axis-0 stencil reach (upwind2, 21/81-point)

typedef int (*HostAllgather)(const void* send, void* recv, long long nbytes);
typedef int (*HostSendrecv)(const void* send, long long sbytes, int dst, void* recv, long long rbytes, int src);
typedef int (*HostBcast)(void* buf, long long nbytes, int root);

struct Comm {
  int rank = 0, size = 1;
  int kind = 0;  // 1 NCCL, 2 host callbacks
  HostAllgather h_allgather = nullptr;
  HostSendrecv h_sendrecv = nullptr;
  HostBcast h_bcast = nullptr;
  void* nccl = nullptr;  // ncclComm_t
  DistRed red{};         // reduction plumbing (LaunchCfg::dist of distributed levels)

  bool graphable() const { return kind == 1; }
  // stream-ordered collectives on device buffers
  void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t s);
  void bcast(void* dbuf, size_t bytes, int root, cudaStream_t s);
  // fill the h planes below and above the owned block of v (v points at the first owned plane)
  void halo(void* v, size_t plane_bytes, int nown, int h, cudaStream_t s);
  void group_start();
  void group_end();
  // host-side: OR / MAX of small host arrays across ranks (setup decisions)
  void allreduce_or_u64(unsigned long long* v, int n, cudaStream_t s);

 private:
  void* hstage = nullptr;
  size_t hstage_bytes = 0;
  void* dscratch = nullptr;
  char* stage(size_t bytes);
};

Comm* dist_comm();  // null unless a distributed context is active
extern int g_dist_min_planes;  // a coarse level stays distributed while every slab keeps >= this many planes
extern int g_dist_levels;      // > 0: distribute exactly this many levels (tests / tuning)
extern double g_dist_min_work;  // split a coarse level while points x planes >= this x R/(R-1) (cost model)
int dist_init_nccl(int rank, int size, const char* unique_id /* 128 bytes */);
int dist_nccl_unique_id(char* out /* 128 bytes */);
int dist_init_host(int rank, int size, HostAllgather ag, HostSendrecv sr, HostBcast bc);
void dist_finalize();

// Slab boundaries of the fine axis: size + 1 entries, interior boundaries multiples of `align`
// (so every distributed coarse level's slabs nest: boundary >> l); empty when impossible.
std::vector<int> slab_bounds(int n1, int size, int align);

}  // namespace hadr
