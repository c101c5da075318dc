// Precompiled sm_100a kernels: ordered reduction combine, opaque builtins,
// fills and rect pack/unpack for transfers.
//
// Builtins restate diffusekit executor.py:93-113 on the GPU:
//   MATVEC / SPMV (dense a2 = a0 @ a1)  -- one warp per output row
//   NORM  (a1 += sum(a0 * a0))          -- deterministic two-level tree
//   OPAQUE (W/RW args += 1.0)
// plus the new SPMV_CSR kind: per row, acc = 0.0 then
// acc = acc + vals[j] * x[cols[j]] left to right -- bit-identical to the
// oracle's definition because the order and the roundings are the same and
// __dmul_rn/__dadd_rn forbid FMA contraction.

#include <string>

#include "dk_internal.h"

namespace dk {

struct VIdx {
  // element offset of the i-th element (row-major order) of a view
  __device__ static int64_t off(const dk_view& v, int64_t i) {
    int64_t o = 0;
    for (int d = v.rank - 1; d >= 0; --d) {
      int64_t e = v.ext[d];
      o += (i % e) * v.stride[d];
      i /= e;
    }
    return o;
  }
};

__global__ void k_accum(dk_view t, const double* __restrict__ vals, int64_t stride, int nvals) {
  int64_t n = 1;
  for (int d = 0; d < t.rank; ++d) n *= t.ext[d];
  double* p = (double*)t.ptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double* q = p + VIdx::off(t, i);
    double a = *q;
    for (int k = 0; k < nvals; ++k) a = __dadd_rn(a, vals[k * stride]);
    *q = a;
  }
}

void launch_accum(const dk_view& target, const double* vals, int64_t stride, int nvals, cudaStream_t s) {
  int64_t n = view_volume(target);
  if (n == 0) return;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
  k_accum<<<blocks, 256, 0, s>>>(target, vals, stride, nvals);
  DK_CUDA(cudaGetLastError());
  st().launches++;
}

__global__ void k_fill(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_timestamp(unsigned long long* buf, int64_t idx) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  buf[idx] = t;
}

void launch_timestamp(uint64_t buf, int64_t idx, cudaStream_t s) {
  k_timestamp<<<1, 1, 0, s>>>((unsigned long long*)buf, idx);
  DK_CUDA(cudaGetLastError());
}

void launch_fill(double* p, int64_t n, double value, cudaStream_t s) {
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)st().sm_count * 8);
  k_fill<<<blocks, 256, 0, s>>>(p, n, value);
  DK_CUDA(cudaGetLastError());
  st().launches++;
}

// pack a strided view into a dense buffer (unpack: the reverse); 8-byte elements
__global__ void k_pack(dk_view v, double* buf, int unpack) {
  int64_t n = 1;
  for (int d = 0; d < v.rank; ++d) n *= v.ext[d];
  double* p = (double*)v.ptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = VIdx::off(v, i);
    if (unpack)
      p[o] = buf[i];
    else
      buf[i] = p[o];
  }
}

void launch_pack(const dk_view& src, double* dst, cudaStream_t s, bool unpack) {
  int64_t n = view_volume(src);
  if (n == 0) return;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)st().sm_count * 8);
  k_pack<<<blocks, 256, 0, s>>>(src, dst, unpack ? 1 : 0);
  DK_CUDA(cudaGetLastError());
  st().launches++;
}

// ---- SPMV_CSR ---------------------------------------------------------------

template <class I>
__global__ void __launch_bounds__(256) k_spmv_csr(const I* __restrict__ rowptr, const I* __restrict__ cols,
                                                  const double* __restrict__ vals, const double* __restrict__ x,
                                                  double* __restrict__ y, int64_t nrows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = (int64_t)rowptr[i], e = (int64_t)rowptr[i + 1];
    double acc = 0.0;
    for (int64_t j = b; j < e; ++j) acc = __dadd_rn(acc, __dmul_rn(__ldg(vals + j), __ldg(x + (int64_t)cols[j])));
    y[i] = acc;
  }
}

// ---- SPMV_CSR, bulk-copy pipeline (int32 indices) ----------------------------
// Persistent CTAs of R/32 consumer warps + 1 producer warp.  The matrix is cut
// into chunks of R rows; chunk c's rowptr slab and its contiguous nonzero
// slab [rowptr[r0], rowptr[r1]) of vals and cols are moved into a shared-memory
// stage by three cp.async.bulk copies (16-byte-rounded ranges: rounding never
// leaves the 2 MiB granule a view lies in) completing on the stage's full
// mbarrier; consumers release the stage on its empty mbarrier.  Two
// stages per CTA, four CTAs per SM: ~100 KB of the nonzero stream in flight
// per SM without per-thread dependent loads, and 32 consumer warps per SM to
// hide the x gathers.  Each consumer thread then sums one
// row from shared memory: acc = 0.0; acc = acc + vals[j] * x[cols[j]] left
// to right with __dmul_rn / __dadd_rn -- the same order and roundings as the
// oracle's definition, so the result is bit-identical to k_spmv_csr.  A chunk
// whose nonzeros exceed the stage capacity is flagged and read from global.
// Optional epilogue (dot != nullptr): per-CTA partial of sum_i p[i] * y[i]
// over the tile's rows (p = x at row offset x_row0), for the opt-in SpMV +
// partial-dot fusion; per-thread in row order, then a fixed warp / CTA tree.
namespace {
template <int R, int CAP, int S>
struct __align__(16) SpStageT {
  double vals[CAP + 2];
  int32_t cols[CAP + 4];
  int32_t rowptr[R + 8];
  int64_t rp0;
  int32_t voff, coff, roff, mode;
};
template <int R, int CAP, int S>
struct SpSharedT {
  SpStageT<R, CAP, S> st[S];
  unsigned long long full[S], empty[S];
  double red[R / 32];
  int last;  // dot epilogue: this CTA folds the partials
};
__device__ __forceinline__ uint32_t sp_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void sp_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void sp_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
}  // namespace

// R rows per chunk (one per consumer thread), CAP nonzeros per stage, S stages, MINB CTAs per SM
template <int R, int CAP, int S, int MINB>
__global__ void __launch_bounds__(R + 32, MINB)
    k_spmv_csr_bulk(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                    const double* __restrict__ vals, const double* __restrict__ x, double* __restrict__ y,
                    int64_t nrows, double* __restrict__ dot, int64_t x_row0) {
  constexpr int NC = R / 32;  // consumer warps
  extern __shared__ __align__(16) unsigned char sp_raw[];
  SpSharedT<R, CAP, S>& SH = *reinterpret_cast<SpSharedT<R, CAP, S>*>(sp_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = (nrows + R - 1) / R;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sp_smem(&SH.full[s])), "r"(1) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sp_smem(&SH.empty[s])), "r"(NC) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NC) {  // producer
    if (lane == 0) {
      int64_t c = blockIdx.x;
      int64_t nr0 = 0, nr1 = 0;
      if (c < nchunks) {
        nr0 = __ldg(rowptr + c * R);
        nr1 = __ldg(rowptr + (c * R + R < nrows ? c * R + R : nrows));
      }
      for (int64_t k = 0; c < nchunks; c += gridDim.x, ++k) {
        const int s = (int)(k % S);
        if (k >= S) sp_wait(sp_smem(&SH.empty[s]), (uint32_t)(((k / S) - 1) & 1));
        const int64_t r0 = c * R, r1 = (r0 + R < nrows ? r0 + R : nrows);
        const int64_t rp0 = nr0, rp1 = nr1;
        // prefetch the next chunk's boundaries (consumed one iteration later)
        const int64_t cn = c + gridDim.x;
        if (cn < nchunks) {
          nr0 = __ldg(rowptr + cn * R);
          nr1 = __ldg(rowptr + (cn * R + R < nrows ? cn * R + R : nrows));
        }
        SpStageT<R, CAP, S>& st = SH.st[s];
        st.rp0 = rp0;
        const uint32_t fb = sp_smem(&SH.full[s]);
        if (rp1 - rp0 <= CAP) {
          const uintptr_t va = (uintptr_t)(vals + rp0) & ~(uintptr_t)15, vb = ((uintptr_t)(vals + rp1) + 15) & ~(uintptr_t)15;
          const uintptr_t ca = (uintptr_t)(cols + rp0) & ~(uintptr_t)15, cb = ((uintptr_t)(cols + rp1) + 15) & ~(uintptr_t)15;
          const uintptr_t ra = (uintptr_t)(rowptr + r0) & ~(uintptr_t)15, rb = ((uintptr_t)(rowptr + r1 + 1) + 15) & ~(uintptr_t)15;
          st.voff = (int32_t)(((uintptr_t)(vals + rp0) - va) / 8);
          st.coff = (int32_t)(((uintptr_t)(cols + rp0) - ca) / 4);
          st.roff = (int32_t)(((uintptr_t)(rowptr + r0) - ra) / 4);
          st.mode = 0;
          const uint32_t vbytes = (uint32_t)(vb - va), cbytes = (uint32_t)(cb - ca), rbytes = (uint32_t)(rb - ra);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                       :: "r"(fb), "r"(vbytes + cbytes + rbytes) : "memory");
          sp_bulk(sp_smem(st.rowptr), (const void*)ra, rbytes, fb);
          if (vbytes) sp_bulk(sp_smem(st.vals), (const void*)va, vbytes, fb);
          if (cbytes) sp_bulk(sp_smem(st.cols), (const void*)ca, cbytes, fb);
        } else {
          st.mode = 1;  // too many nonzeros for a stage: consumers read this chunk from global
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(fb) : "memory");
        }
      }
    }
    return;
  }
  // consumers: one row per thread per chunk
  double dacc = 0.0;
  for (int64_t c = blockIdx.x, k = 0; c < nchunks; c += gridDim.x, ++k) {
    const int s = (int)(k % S);
    sp_wait(sp_smem(&SH.full[s]), (uint32_t)((k / S) & 1));
    const SpStageT<R, CAP, S>& st = SH.st[s];
    const int64_t row = c * R + threadIdx.x;
    if (row < nrows) {
      double acc = 0.0;
      if (st.mode == 0) {
        const int b = (int)(st.rowptr[st.roff + threadIdx.x] - st.rp0);
        const int e = (int)(st.rowptr[st.roff + threadIdx.x + 1] - st.rp0);
        const double* sv = st.vals + st.voff;
        const int32_t* sc = st.cols + st.coff;
        for (int j = b; j < e; j += 8) {
          const int len = e - j;
          double xv[8];
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < len) xv[t] = __ldg(x + sc[j + t]);
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < len) acc = __dadd_rn(acc, __dmul_rn(sv[j + t], xv[t]));
        }
      } else {
        const int64_t b = rowptr[row], e = rowptr[row + 1];
        for (int64_t j = b; j < e; ++j) acc = __dadd_rn(acc, __dmul_rn(__ldg(vals + j), __ldg(x + cols[j])));
      }
      y[row] = acc;
      if (dot) dacc = __dadd_rn(dacc, __dmul_rn(__ldg(x + x_row0 + row), acc));
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sp_smem(&SH.empty[s])) : "memory");
  }
  if (dot) {
    for (int o = 16; o; o >>= 1) dacc = __dadd_rn(dacc, __shfl_xor_sync(0xffffffffu, dacc, o));
    if (lane == 0) SH.red[warp] = dacc;
    asm volatile("bar.sync 1, %0;" :: "r"(R) : "memory");  // consumers only
    unsigned* ticket = reinterpret_cast<unsigned*>(dot + DK_SPMV_DOT_PARTS);
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < NC; ++w) t = __dadd_rn(t, SH.red[w]);
      dot[blockIdx.x] = t;
      __threadfence();
      SH.last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    asm volatile("bar.sync 1, %0;" :: "r"(R) : "memory");
    if (SH.last) {
      // the last CTA folds the per-CTA partials: strided in-order sums, then a fixed
      // shuffle + warp-order tree (the grid depends only on nrows: run-to-run identical)
      __threadfence();
      double t = 0.0;
      for (int i = threadIdx.x; i < (int)gridDim.x; i += R) t = __dadd_rn(t, __ldcg(dot + i));
      for (int o = 16; o; o >>= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
      if (lane == 0) SH.red[warp] = t;
      asm volatile("bar.sync 1, %0;" :: "r"(R) : "memory");
      if (threadIdx.x == 0) {
        double u = 0.0;
        for (int w = 0; w < NC; ++w) u = __dadd_rn(u, SH.red[w]);
        dot[DK_SPMV_DOT_TOTAL] = u;
        *ticket = 0u;  // left zero for the buffer's next use
      }
    }
  }
}

// launch configurations (DK_SPMV_CFG selects one; default 0)
struct SpCfg {
  void (*fn)(const int32_t*, const int32_t*, const double*, const double*, double*, int64_t, double*, int64_t);
  int rows, threads, smem, minb;
};
template <int R, int CAP, int S, int MINB>
static SpCfg sp_cfg() {
  SpCfg c;
  c.fn = k_spmv_csr_bulk<R, CAP, S, MINB>;
  c.rows = R;
  c.threads = R + 32;
  c.smem = (int)sizeof(SpSharedT<R, CAP, S>);
  c.minb = MINB;
  cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem);
  return c;
}
static const SpCfg& spmv_cfg() {
  static const SpCfg cfg = [] {
    const char* e = getenv("DK_SPMV_CFG");
    const int v = e ? atoi(e) : 0;
    switch (v) {
      // measured at 67M rows (B200, bench cg): 1: 1.040 ms, 2: 0.778, 3: 0.784, 4: 0.858, 5: 1.301;
      // the thread-per-row kernel (DK_SPMV_SIMPLE) 0.866.  Occupancy (4 CTAs = 32 consumer warps
      // per SM to hide the x gathers) matters more than stage depth.
      case 1: return sp_cfg<256, 2048, 4, 2>();
      case 3: return sp_cfg<512, 3072, 2, 2>();
      case 4: return sp_cfg<256, 1536, 3, 3>();
      case 5: return sp_cfg<128, 768, 4, 6>();
      default: return sp_cfg<256, 1536, 2, 4>();
    }
  }();
  return cfg;
}

// ---- dense matvec: one warp per row, fixed lane order ------------------------

__global__ void k_matvec(dk_view A, dk_view xv, dk_view yv) {
  const int64_t m = A.ext[0], k = A.ext[1];
  const double* a = (const double*)A.ptr;
  const double* x = (const double*)xv.ptr;
  double* y = (double*)yv.ptr;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = warp; row < m; row += nw) {
    double acc = 0.0;
    for (int64_t j = lane; j < k; j += 32)
      acc = __dadd_rn(acc, __dmul_rn(a[row * A.stride[0] + j * A.stride[1]], x[j * xv.stride[0]]));
    for (int o = 16; o; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) y[row * yv.stride[0]] = acc;
  }
}

// ---- NORM: target += sum(x*x) --------------------------------------------------
// Grid-wide and deterministic: CTA b sums its contiguous element range
// (thread-strided, warp shuffle tree, fixed smem tree) into parts[b]; one
// thread then folds parts[0..G) in order and adds the total.  G depends only
// on n and the SM count.

__global__ void __launch_bounds__(256) k_norm_part(dk_view xv, double* parts, int64_t per_cta) {
  __shared__ double sh[8];
  int64_t n = 1;
  for (int d = 0; d < xv.rank; ++d) n *= xv.ext[d];
  const double* x = (const double*)xv.ptr;
  const int64_t lo = (int64_t)blockIdx.x * per_cta, hi = lo + per_cta < n ? lo + per_cta : n;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double v = x[VIdx::off(xv, i)];
    acc = __dadd_rn(acc, __dmul_rn(v, v));
  }
  for (int o = 16; o; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s = __dadd_rn(s, sh[w]);
    parts[blockIdx.x] = s;
  }
}

__global__ void k_norm_fold(dk_view t, const double* parts, int nparts) {
  double s = 0.0;
  for (int b = 0; b < nparts; ++b) s = __dadd_rn(s, parts[b]);
  int64_t nt = 1;
  for (int d = 0; d < t.rank; ++d) nt *= t.ext[d];
  double* tp = (double*)t.ptr;
  for (int64_t i = 0; i < nt; ++i) {
    double* q = tp + VIdx::off(t, i);
    *q = __dadd_rn(*q, s);
  }
}

// single-block variant (DK_NORM_ONEBLOCK=1): round 1's kernel

__global__ void k_norm(dk_view xv, dk_view t) {
  __shared__ double sh[32];
  int64_t n = 1;
  for (int d = 0; d < xv.rank; ++d) n *= xv.ext[d];
  const double* x = (const double*)xv.ptr;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double v = x[VIdx::off(xv, i)];
    acc = __dadd_rn(acc, __dmul_rn(v, v));
  }
  for (int o = 16; o; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = __dadd_rn(s, sh[w]);
    int64_t nt = 1;
    for (int d = 0; d < t.rank; ++d) nt *= t.ext[d];
    double* tp = (double*)t.ptr;
    for (int64_t i = 0; i < nt; ++i) {
      double* q = tp + VIdx::off(t, i);
      *q = __dadd_rn(*q, s);
    }
  }
}

__global__ void k_add_one(dk_view v) {
  int64_t n = 1;
  for (int d = 0; d < v.rank; ++d) n *= v.ext[d];
  double* p = (double*)v.ptr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double* q = p + VIdx::off(v, i);
    *q = __dadd_rn(*q, 1.0);
  }
}

static void check_f64(const dk_view& v, const char* what) {
  if (v.dtype != DK_F64) fail(DK_ERR_UNSUPPORTED, "%s: expected an f64 view", what);
}

int launch_spmv_csr_dot(const dk_view* v, double* parts, int64_t x_row0, cudaStream_t s) {
  const dk_view &rp = v[0], &cl = v[1], &vl = v[2], &x = v[3], &y = v[4];
  check_f64(vl, "SPMV_CSR vals");
  check_f64(x, "SPMV_CSR x");
  check_f64(y, "SPMV_CSR y");
  if (rp.dtype != DK_I32 || cl.dtype != DK_I32) fail(DK_ERR_UNSUPPORTED, "SPMV_CSR+dot needs int32 indices");
  if (x.rank != 1 || y.rank != 1 || x.stride[0] != 1 || y.stride[0] != 1)
    fail(DK_ERR_UNSUPPORTED, "SPMV_CSR+dot needs contiguous rank-1 x and y");
  const int64_t nrows = view_volume(y);
  if (view_volume(rp) != nrows + 1) fail(DK_ERR_ARG, "SPMV_CSR: rowptr has %lld entries for %lld rows",
                                         (long long)view_volume(rp), (long long)nrows);
  if (x_row0 < 0 || x_row0 + nrows > x.ext[0]) fail(DK_ERR_ARG, "SPMV_CSR+dot: x rows out of range");
  if (nrows == 0) return 0;
  const SpCfg& cfg = spmv_cfg();
  const int64_t nchunks = (nrows + cfg.rows - 1) / cfg.rows;
  const int blocks = (int)std::min<int64_t>(std::min<int64_t>(nchunks, (int64_t)st().sm_count * cfg.minb), DK_SPMV_DOT_PARTS);
  cfg.fn<<<blocks, cfg.threads, cfg.smem, s>>>((const int32_t*)rp.ptr, (const int32_t*)cl.ptr,
                                               (const double*)vl.ptr, (const double*)x.ptr, (double*)y.ptr, nrows,
                                               parts, x_row0);
  DK_CUDA(cudaGetLastError());
  st().launches++;
  return blocks;
}

void launch_builtin(const std::string& kind, const dk_view* v, int n, const int32_t* writes, cudaStream_t s) {
  const int sms = st().sm_count;
  if (kind == "SPMV_CSR") {
    if (n != 5) fail(DK_ERR_ARG, "SPMV_CSR expects 5 args, got %d", n);
    const dk_view &rp = v[0], &cl = v[1], &vl = v[2], &x = v[3], &y = v[4];
    check_f64(vl, "SPMV_CSR vals");
    check_f64(x, "SPMV_CSR x");
    check_f64(y, "SPMV_CSR y");
    if (rp.dtype != cl.dtype) fail(DK_ERR_UNSUPPORTED, "SPMV_CSR rowptr/cols dtypes differ");
    for (int i = 0; i < 5; ++i)
      if (v[i].rank > 1 && view_volume(v[i]) > 0) {
        // only contiguous rank-1 segments are supported (row-band tiles)
        for (int d = 0; d + 1 < v[i].rank; ++d)
          if (v[i].ext[d] != 1) fail(DK_ERR_UNSUPPORTED, "SPMV_CSR arg %d is not a contiguous segment", i);
      }
    const int64_t nrows = view_volume(y);
    if (view_volume(rp) != nrows + 1 && !(nrows == 0 && view_volume(rp) <= 1))
      fail(DK_ERR_ARG, "SPMV_CSR: rowptr has %lld entries for %lld rows", (long long)view_volume(rp), (long long)nrows);
    if (nrows == 0) return;
    // one CTA per 256 rows (no persistent grid-stride loop): as for the JIT's
    // streaming nests, a grid covering the whole matrix keeps the HBM stream
    // tighter (0.862 vs 0.875 ms at 67M rows; DK_SPMV_PERSIST restores the
    // persistent grid).  Staging each CTA's nonzeros in shared memory first
    // was measured slower (1.17 ms), and so were loading each row in predicated
    // chunks of 8 (cols, vals, then the x gathers: 1.62 ms) and a
    // warp-cooperative layout (coalesced vals/cols over the warp's 32 rows,
    // products staged in shared memory, per-row in-order sums: 1.46 ms).
    // The per-row loop's strided loads are served from L1 (67 % hits).
    static const bool persist = getenv("DK_SPMV_PERSIST") != nullptr;
    static const bool simple = getenv("DK_SPMV_SIMPLE") != nullptr;
    if (rp.dtype == DK_I32 && !simple && !persist && nrows >= 4096) {
      const SpCfg& cfg = spmv_cfg();
      const int64_t nchunks = (nrows + cfg.rows - 1) / cfg.rows;
      const int blocks = (int)std::min<int64_t>(nchunks, (int64_t)sms * cfg.minb);
      cfg.fn<<<blocks, cfg.threads, cfg.smem, s>>>((const int32_t*)rp.ptr, (const int32_t*)cl.ptr,
                                                   (const double*)vl.ptr, (const double*)x.ptr, (double*)y.ptr,
                                                   nrows, nullptr, 0);
      DK_CUDA(cudaGetLastError());
      st().launches++;
      return;
    }
    const int blocks = (int)std::min<int64_t>((nrows + 255) / 256, persist ? (int64_t)sms * 8 : 0x7fffffff);
    if (rp.dtype == DK_I32)
      k_spmv_csr<int32_t><<<blocks, 256, 0, s>>>((const int32_t*)rp.ptr, (const int32_t*)cl.ptr,
                                                  (const double*)vl.ptr, (const double*)x.ptr, (double*)y.ptr, nrows);
    else
      k_spmv_csr<double><<<blocks, 256, 0, s>>>((const double*)rp.ptr, (const double*)cl.ptr,
                                                 (const double*)vl.ptr, (const double*)x.ptr, (double*)y.ptr, nrows);
    DK_CUDA(cudaGetLastError());
    st().launches++;
    return;
  }
  if (kind == "MATVEC" || kind == "SPMV") {
    if (n != 3) fail(DK_ERR_ARG, "%s expects 3 args", kind.c_str());
    for (int i = 0; i < 3; ++i) check_f64(v[i], kind.c_str());
    if (v[0].rank != 2 || v[1].rank != 1 || v[2].rank != 1 || v[0].ext[1] != v[1].ext[0] || v[0].ext[0] != v[2].ext[0])
      fail(DK_ERR_UNSUPPORTED, "%s: only (m,k) @ (k,) -> (m,) is supported", kind.c_str());
    const int64_t m = v[0].ext[0];
    if (m == 0) return;
    int blocks = (int)std::min<int64_t>((m * 32 + 255) / 256, (int64_t)sms * 8);
    k_matvec<<<blocks, 256, 0, s>>>(v[0], v[1], v[2]);
    DK_CUDA(cudaGetLastError());
    st().launches++;
    return;
  }
  if (kind == "NORM") {
    if (n != 2) fail(DK_ERR_ARG, "NORM expects 2 args");
    check_f64(v[0], "NORM");
    check_f64(v[1], "NORM");
    static const bool one = getenv("DK_NORM_ONEBLOCK") != nullptr;
    const int64_t cnt = view_volume(v[0]);
    if (one || cnt < (1 << 16)) {
      k_norm<<<1, 1024, 0, s>>>(v[0], v[1]);
      DK_CUDA(cudaGetLastError());
      st().launches++;
      return;
    }
    const int64_t want = (cnt + 256 * 16 - 1) / (256 * 16);
    const int g = (int)std::min<int64_t>(want, (int64_t)sms * 4);
    const int64_t per = (cnt + g - 1) / g;
    double* parts = nullptr;
    DK_CUDA(cudaMallocAsync((void**)&parts, sizeof(double) * g, s));
    k_norm_part<<<g, 256, 0, s>>>(v[0], parts, per);
    DK_CUDA(cudaGetLastError());
    k_norm_fold<<<1, 1, 0, s>>>(v[1], parts, g);
    DK_CUDA(cudaGetLastError());
    DK_CUDA(cudaFreeAsync(parts, s));
    st().launches += 2;
    return;
  }
  if (kind == "OPAQUE") {
    for (int i = 0; i < n; ++i) {
      if (!writes[i]) continue;
      check_f64(v[i], "OPAQUE");
      int64_t cnt = view_volume(v[i]);
      if (cnt == 0) continue;
      int blocks = (int)std::min<int64_t>((cnt + 255) / 256, (int64_t)sms * 8);
      k_add_one<<<blocks, 256, 0, s>>>(v[i]);
      DK_CUDA(cudaGetLastError());
      st().launches++;
    }
    return;
  }
  fail(DK_ERR_STATE, "no builtin for task kind '%s'", kind.c_str());
}

}  // namespace dk
