// Copy-pattern microbenchmark (diagnostic): persistent grid-stride vs one-shot
// grids, flat vs 2-D interior rows, for the stencil COPY's layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o copybench copybench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

// flat: n pairs, persistent grid-stride, U pairs per thread per step
template <int U>
__global__ void __launch_bounds__(256) flat_persist(const double2* __restrict__ s, double2* __restrict__ d, int64_t n) {
  for (int64_t q0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; q0 < n; q0 += (int64_t)gridDim.x * 256 * U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (q0 + u * 256 < n) v[u] = s[q0 + u * 256];
#pragma unroll
    for (int u = 0; u < U; ++u) if (q0 + u * 256 < n) d[q0 + u * 256] = v[u];
  }
}
// flat one-shot: each thread U pairs, grid covers everything
template <int U>
__global__ void __launch_bounds__(256) flat_once(const double2* __restrict__ s, double2* __restrict__ d, int64_t n) {
  const int64_t q0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x;
  double2 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) if (q0 + u * 256 < n) v[u] = s[q0 + u * 256];
#pragma unroll
  for (int u = 0; u < U; ++u) if (q0 + u * 256 < n) d[q0 + u * 256] = v[u];
}
// 2-D interior: dst row r starts at dst + (r+1)*ld + 1 (8-byte stores), src rows of w (aligned)
template <int U>
__global__ void __launch_bounds__(256) rows_persist(const double* __restrict__ s, double* __restrict__ d, int64_t rows,
                                                     int64_t w, int64_t ld) {
  const int64_t np = (w + 1) / 2;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const double* sr = s + r * w;
    double* dr = d + (r + 1) * ld + 1;
    for (int64_t q0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; q0 < np; q0 += (int64_t)gridDim.x * 256 * U) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { int64_t q = q0 + u * 256; if (q < np) v[u] = *reinterpret_cast<const double2*>(sr + 2 * q); }
#pragma unroll
      for (int u = 0; u < U; ++u) { int64_t q = q0 + u * 256; if (q < np) { dr[2 * q] = v[u].x; dr[2 * q + 1] = v[u].y; } }
    }
  }
}
template <int U>
__global__ void __launch_bounds__(256) rows_once(const double* __restrict__ s, double* __restrict__ d, int64_t rows,
                                                  int64_t w, int64_t ld) {
  const int64_t np = (w + 1) / 2;
  const int64_t r = blockIdx.y;
  const double* sr = s + r * w;
  double* dr = d + (r + 1) * ld + 1;
  const int64_t q0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x;
  double2 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { int64_t q = q0 + u * 256; if (q < np) v[u] = *reinterpret_cast<const double2*>(sr + 2 * q); }
#pragma unroll
  for (int u = 0; u < U; ++u) { int64_t q = q0 + u * 256; if (q < np) { dr[2 * q] = v[u].x; dr[2 * q + 1] = v[u].y; } }
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int i = 0; i < 8; ++i) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const int64_t n = 32768, w = n - 2, rows = n - 2;
  double *g, *wk;
  CK(cudaMalloc(&g, n * n * 8));
  CK(cudaMalloc(&wk, w * rows * 8));
  cudaMemset(g, 0, n * n * 8); cudaMemset(wk, 0, w * rows * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = 16.0 * w * rows;
  const int64_t fp = w * rows / 2;
  auto rep = [&](const char* name, float ms) { printf("%-34s %.3f ms  %.0f GB/s\n", name, ms, bytes / ms / 1e6); };
  for (int occ : {4, 8}) {
    char nm[64];
    snprintf(nm, 64, "flat persist U2 occ%d", occ);
    rep(nm, timeit([&] { flat_persist<2><<<sms * occ, 256>>>((const double2*)wk, (double2*)g, fp); }));
    snprintf(nm, 64, "flat persist U4 occ%d", occ);
    rep(nm, timeit([&] { flat_persist<4><<<sms * occ, 256>>>((const double2*)wk, (double2*)g, fp); }));
  }
  rep("flat once U2", timeit([&] { flat_once<2><<<(unsigned)((fp + 511) / 512), 256>>>((const double2*)wk, (double2*)g, fp); }));
  rep("flat once U4", timeit([&] { flat_once<4><<<(unsigned)((fp + 1023) / 1024), 256>>>((const double2*)wk, (double2*)g, fp); }));
  const int64_t np = (w + 1) / 2;
  for (int occ : {4, 8}) {
    const int gx = (int)((np + 511) / 512), gy = sms * occ / gx;
    char nm[64];
    snprintf(nm, 64, "rows persist U2 occ%d (%dx%d)", occ, gx, gy);
    rep(nm, timeit([&] { rows_persist<2><<<dim3(gx, gy), 256>>>(wk, g, rows, w, n); }));
  }
  rep("rows once U2", timeit([&] { rows_once<2><<<dim3((unsigned)((np + 511) / 512), (unsigned)rows), 256>>>(wk, g, rows, w, n); }));
  rep("rows once U4", timeit([&] { rows_once<4><<<dim3((unsigned)((np + 1023) / 1024), (unsigned)rows), 256>>>(wk, g, rows, w, n); }));
  CK(cudaGetLastError());
  return 0;
}
