// Microbenchmark of synchronisation primitives on B200 (sm_100a):
//  1. back-to-back dependent tiny kernels in a CUDA graph (per-node latency)
//  2. tiny kernels with a last-block grid reduction (our current pattern)
//  3. persistent cooperative kernel: flat grid barrier (one atomic per CTA)
//  4. persistent kernel: hierarchical barrier (cluster barrier + one atomic per cluster)
//  5. cluster barrier alone (barrier.cluster.arrive/wait) inside one cluster
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o sync_mb tools/sync_microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

__global__ void k_tiny(int* p) {
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}

__global__ void k_red(double* part, unsigned* ticket, double* out, int n) {
  __shared__ double sm[32];
  double v = threadIdx.x + blockIdx.x;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) {
    double t = 0;
    for (int i = 0; i < blockDim.x / 32; ++i) t += sm[i];
    part[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    double t = 0;
    for (int i = 0; i < gridDim.x; ++i) t += ((volatile double*)part)[i];
    *out = t;
    *ticket = 0;
  }
}

__device__ __forceinline__ void flat_barrier(unsigned* count, unsigned* gen, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g = *(volatile unsigned*)gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nb - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*(volatile unsigned*)gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_persist_flat(unsigned* count, unsigned* gen, int iters, double* out) {
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    flat_barrier(count, gen, gridDim.x);
    acc += i;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

__device__ __forceinline__ void cluster_sync_hw() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void k_persist_hier(unsigned* count, unsigned* gen, int iters, double* out) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned nclusters = gridDim.x / cl.num_blocks();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    cluster_sync_hw();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
      unsigned g = *(volatile unsigned*)gen;
      __threadfence();
      if (atomicAdd(count, 1u) == nclusters - 1) {
        *count = 0;
        __threadfence();
        atomicAdd(gen, 1u);
      } else {
        while (*(volatile unsigned*)gen == g) {
        }
      }
      __threadfence();
    }
    cluster_sync_hw();
    acc += i;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

__global__ void k_cluster_only(int iters, double* out) {
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    cluster_sync_hw();
    acc += i;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

// DSMEM all-reduce of one double across the cluster + barrier
__global__ void k_cluster_reduce(int iters, double* out) {
  __shared__ double slot[2];
  cg::cluster_group cl = cg::this_cluster();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) slot[i & 1] = i + cl.block_rank();
    cluster_sync_hw();
    double t = 0;
    if (threadIdx.x < cl.num_blocks()) {
      double* r = cl.map_shared_rank(&slot[i & 1], threadIdx.x);
      t = *r;
    }
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    acc += t;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

int main() {
  int dev = 0, nsm = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  int* p;
  double *part, *out;
  unsigned *ticket, *cnt, *gen;
  CK(cudaMalloc(&p, 64));
  CK(cudaMalloc(&part, 8192 * 8));
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&ticket, 64));
  CK(cudaMalloc(&cnt, 64));
  CK(cudaMalloc(&gen, 64));
  CK(cudaMemset(ticket, 0, 64));
  CK(cudaMemset(cnt, 0, 64));
  CK(cudaMemset(gen, 0, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;
  const int NK = 2000;
  for (int grid : {1, 17, 148, 1184}) {
    // graph of NK dependent kernels
    for (int variant = 0; variant < 2; ++variant) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
      for (int i = 0; i < NK; ++i) {
        if (variant == 0)
          k_tiny<<<grid, 256, 0, s>>>(p);
        else
          k_red<<<grid, 256, 0, s>>>(part, ticket, out, 0);
      }
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaStreamSynchronize(s));
      CK(cudaEventRecord(e0, s));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("graph %-10s grid=%5d : %.3f us/kernel\n", variant ? "reduce" : "tiny", grid, ms * 1e3 / NK);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  // persistent flat barrier
  const int IT = 20000;
  for (int grid : {16, 74, 148, 296}) {
    int threads = grid > nsm ? 512 : 1024;
    void* args[] = {&cnt, &gen, (void*)&IT, &out};
    CK(cudaEventRecord(e0, s));
    CK(cudaLaunchCooperativeKernel((void*)k_persist_flat, grid, threads, args, 0, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("flat grid barrier  grid=%4d x %4d : %.3f us/barrier\n", grid, threads, ms * 1e3 / IT);
  }
  // hierarchical (cluster + atomic)
  for (int csz : {4, 8, 16}) {
    for (int grid : {csz, 144, 148}) {
      if (grid % csz) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(1024);
      cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csz;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      if (csz > 8) {
        CK(cudaFuncSetAttribute(k_persist_hier, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(k_cluster_only, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        CK(cudaFuncSetAttribute(k_cluster_reduce, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      }
      int ncl = 0;
      cudaOccupancyMaxActiveClusters(&ncl, (void*)k_persist_hier, &cfg);
      if (ncl * csz < grid) {
        printf("cluster %d: only %d clusters co-resident, skip grid %d\n", csz, ncl, grid);
        cudaGetLastError();
        continue;
      }
      CK(cudaEventRecord(e0, s));
      cudaError_t err = cudaLaunchKernelEx(&cfg, k_persist_hier, cnt, gen, IT, out);
      if (err != cudaSuccess) {
        printf("hier launch failed csz=%d grid=%d: %s\n", csz, grid, cudaGetErrorString(err));
        cudaGetLastError();
        continue;
      }
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("hier barrier cluster=%2d grid=%4d : %.3f us/barrier (max clusters %d)\n", csz, grid, ms * 1e3 / IT, ncl);
      if (grid == csz) {
        cfg.numAttrs = 1;
        CK(cudaEventRecord(e0, s));
        CK(cudaLaunchKernelEx(&cfg, k_cluster_only, IT, out));
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("cluster-only barrier size=%2d : %.3f us/barrier\n", csz, ms * 1e3 / IT);
        CK(cudaEventRecord(e0, s));
        CK(cudaLaunchKernelEx(&cfg, k_cluster_reduce, IT, out));
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("cluster DSMEM allreduce size=%2d : %.3f us/op\n", csz, ms * 1e3 / IT);
      }
    }
  }
  printf("done\n");
  return 0;
}
