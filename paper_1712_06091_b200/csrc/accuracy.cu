// Accuracy workflow on the device:
//   relative_error_map  (helmadr/grid.py:175-191)
//   accuracy_compare    (helmadr/drivers.py:176-196) — masked median / p95 / max
// The error map is one streaming pass (|u - u_ref| / max(|u_ref|, floor)); the
// masked order statistics compact the mask on the device (cub select) and
// radix-sort the surviving errors (non-negative doubles), so only the few order
// statistics numpy's median / linear percentile need are read back.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_select.cuh>

#include "../../include/hadr.h"
#include "engine.h"

namespace hadr {

namespace {

__global__ void k_abs(long n, const cplx* __restrict__ z, double* __restrict__ out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const cplx v = z[i];
    out[i] = hypot(v.x, v.y);  // numpy |z| = hypot(re, im)
  }
}

// err = |u - ref| / (|ref| < floor ? floor : |ref|); flag = |ref| >= floor
__global__ void k_relerr(long n, const cplx* __restrict__ u, const cplx* __restrict__ ref,
                         const double* __restrict__ refmag, double floor, double* __restrict__ err,
                         unsigned char* __restrict__ flag) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const cplx a = u[i], b = ref[i];
    const double m = refmag[i];
    const double d = m < floor ? floor : m;
    err[i] = hypot(a.x - b.x, a.y - b.y) / d;
    if (flag) flag[i] = m >= floor;
  }
}

int grid_for(long n) {
  long b = (n + 255) / 256;
  const long cap = (long)Ctx::get().nsm * 8;
  return (int)(b < 1 ? 1 : b > cap ? cap : b);
}

}  // namespace

// Device pointers.  floor < 0 selects the default 1e-12 * max|ref|.  err may be
// null (statistics only).  sorted_out (optional, host): receives the count and
// the order statistics the caller asks for through idx[0..nidx).
void accuracy_stats(long n, const cplx* u, const cplx* ref, double floor_in, double* err_dev, double* floor_out,
                    long long* count_out, const long long* idx, int nidx, double* vals_out) {
  Ctx& c = Ctx::get();
  cudaStream_t s = c.stream;
  double* mag = dalloc<double>(n);
  double* err = err_dev ? err_dev : dalloc<double>(n);
  unsigned char* flag = dalloc<unsigned char>(n);
  double* sel = dalloc<double>(n);
  double* srt = dalloc<double>(n);
  long long* cnt = dalloc<long long>(1);
  double* mx = dalloc<double>(1);
  k_abs<<<grid_for(n), 256, 0, s>>>(n, ref, mag);
  HADR_CUDA(cudaGetLastError());
  double floor_v = floor_in;
  size_t tb = 0, tb2 = 0, tb3 = 0;
  HADR_CUDA(cub::DeviceReduce::Max(nullptr, tb, mag, mx, n, s));
  HADR_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, err, flag, sel, cnt, n, s));
  HADR_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb3, sel, srt, n, 0, 64, s));
  size_t tmp_bytes = tb > tb2 ? tb : tb2;
  if (tb3 > tmp_bytes) tmp_bytes = tb3;
  void* tmp = pool_alloc(tmp_bytes ? tmp_bytes : 1);
  if (floor_v < 0) {
    HADR_CUDA(cub::DeviceReduce::Max(tmp, tb, mag, mx, n, s));
    double m = 0;
    HADR_CUDA(cudaMemcpyAsync(&m, mx, sizeof(double), cudaMemcpyDeviceToHost, s));
    c.sync();
    floor_v = 1e-12 * m;
  }
  k_relerr<<<grid_for(n), 256, 0, s>>>(n, u, ref, mag, floor_v, err, flag);
  HADR_CUDA(cudaGetLastError());
  if (floor_out) *floor_out = floor_v;
  if (count_out || nidx > 0) {
    HADR_CUDA(cub::DeviceSelect::Flagged(tmp, tb2, err, flag, sel, cnt, n, s));
    long long m = 0;
    HADR_CUDA(cudaMemcpyAsync(&m, cnt, sizeof(long long), cudaMemcpyDeviceToHost, s));
    c.sync();
    if (count_out) *count_out = m;
    if (nidx > 0 && m > 0) {
      // errors are >= 0 (or NaN): their IEEE bit patterns sort like the values
      HADR_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb3, sel, srt, m, 0, 64, s));
      for (int q = 0; q < nidx; ++q) {
        long long k = idx[q] < 0 ? 0 : idx[q] >= m ? m - 1 : idx[q];
        HADR_CUDA(cudaMemcpyAsync(vals_out + q, srt + k, sizeof(double), cudaMemcpyDeviceToHost, s));
      }
    }
  }
  c.sync();
  pool_free(tmp);
  dfree(mag);
  if (!err_dev) dfree(err);
  dfree(flag);
  dfree(sel);
  dfree(srt);
  dfree(cnt);
  dfree(mx);
}

}  // namespace hadr
