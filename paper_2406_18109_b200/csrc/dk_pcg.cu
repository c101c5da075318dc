// Initial store contents generated on the GPU, bit-identical to the reference
// Heap rule (diffusekit executor.py:57-60):
//     np.random.default_rng([seed, sid]).integers(1, 10, size=shape).astype(np.float64)
// and to the harness's seeded uniform fields (Generator.random()).
//
// numpy's default bit generator is PCG64 (128-bit LCG, XSL-RR output).
// integers(1, 10) on int64 draws 32-bit halves of successive 64-bit outputs
// (low half first) and maps each with Lemire's method: m = x * 9,
// value = 1 + (m >> 32), rejecting the draw when (m mod 2^32) < 4
// (= (2^32 - 9) mod 9); the element then consumes the next draw.
// Rejections are rare (4 / 2^32), so the element -> draw mapping is
//     draw(e) = e + #{rejections consumed by elements before e}.
// dk_pcg64_rejects scans a draw range for rejections (one thread per chunk,
// LCG jump-ahead to the chunk start); the host turns them into breakpoints;
// dk_pcg64_fill lets every thread jump to its segment's first draw and
// generate it, so a rank materialises its own band of a 1e9-element store in
// milliseconds instead of replaying the whole stream on the host.

#include <algorithm>
#include <vector>

#include "dk_internal.h"

namespace dk {

struct U128 {
  uint64_t hi, lo;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

__device__ __forceinline__ U128 pcg_mult() { return U128{0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull}; }

__device__ __forceinline__ U128 pcg_step(U128 s, U128 inc) { return add128(mul128(s, pcg_mult()), inc); }

// state after `delta` more steps (Brown's LCG jump-ahead)
__device__ U128 pcg_advance(U128 s, U128 inc, uint64_t delta) {
  U128 acc_mult{0, 1}, acc_plus{0, 0}, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, s), acc_plus);
}

__device__ __forceinline__ uint64_t pcg_out(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ bool lemire9_reject(uint32_t x) { return ((uint64_t)x * 9ull & 0xffffffffull) < 4ull; }

static const int kRejChunk = 4096;  // 64-bit outputs per scan thread

__global__ void k_pcg_rejects(U128 st, U128 inc, int64_t out_end, int64_t* list, unsigned long long* count,
                              int64_t cap) {
  const int64_t nchunk = (out_end + kRejChunk - 1) / kRejChunk;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunk; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j0 = c * kRejChunk, j1 = min(out_end, j0 + kRejChunk);
    U128 s = pcg_advance(st, inc, (uint64_t)j0 + 1);  // state producing output j0
    for (int64_t j = j0; j < j1; ++j) {
      const uint64_t o = pcg_out(s);
      if (lemire9_reject((uint32_t)o)) {
        unsigned long long k = atomicAdd(count, 1ull);
        if ((int64_t)k < cap) list[k] = 2 * j;
      }
      if (lemire9_reject((uint32_t)(o >> 32))) {
        unsigned long long k = atomicAdd(count, 1ull);
        if ((int64_t)k < cap) list[k] = 2 * j + 1;
      }
      s = pcg_step(s, inc);
    }
  }
}

static const int kSeg = 256;  // elements per fill thread

// rows [r0, r1) x cols [c0, c1) of a row-major store with row length L
__global__ void __launch_bounds__(256) k_pcg_fill(double* base, int64_t L, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                                                 U128 st, U128 inc, int kind, double scale, const int64_t* breaks,
                                                 int64_t nb) {
  const int64_t nseg = (c1 - c0 + kSeg - 1) / kSeg;
  const int64_t total = (r1 - r0) * nseg;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = r0 + g / nseg;
    const int64_t cs = c0 + (g % nseg) * kSeg, ce = min(c1, cs + kSeg);
    const int64_t e0 = row * L + cs;
    double* p = base + e0;
    if (kind == 1) {  // Generator.random(): (next_uint64 >> 11) * 2^-53, one output per element
      U128 s = pcg_advance(st, inc, (uint64_t)e0 + 1);
      for (int64_t e = 0; e < ce - cs; ++e) {
        p[e] = __dmul_rn(__dmul_rn((double)(pcg_out(s) >> 11), 1.1102230246251565e-16), scale);
        s = pcg_step(s, inc);
      }
      continue;
    }
    // integers(1, 10): shift = #breaks < e0 (breaks sorted)
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (breaks[mid] < e0) lo = mid + 1; else hi = mid;
    }
    const int64_t d = e0 + lo;
    U128 s = pcg_advance(st, inc, (uint64_t)(d >> 1) + 1);
    uint64_t o = pcg_out(s);
    int half = (int)(d & 1);
    for (int64_t e = 0; e < ce - cs; ++e) {
      uint64_t m;
      for (;;) {
        const uint32_t x = half ? (uint32_t)(o >> 32) : (uint32_t)o;
        if (half) {
          s = pcg_step(s, inc);
          o = pcg_out(s);
        }
        half ^= 1;
        m = (uint64_t)x * 9ull;
        if ((m & 0xffffffffull) >= 4ull) break;
      }
      p[e] = 1.0 + (double)(m >> 32);
    }
  }
}

static U128 u128_of(const uint64_t* v) { return U128{v[0], v[1]}; }

}  // namespace dk

using namespace dk;

extern "C" {

int dk_pcg64_rejects(const uint64_t* state, const uint64_t* inc, int64_t draw_end, int64_t* out, int64_t cap,
                     int64_t* count) {
  return guard([&] {
    require_init();
    cudaStream_t s = st().stream;
    const int64_t out_end = (draw_end + 1) / 2;
    int64_t* dl = nullptr;
    unsigned long long* dc = nullptr;
    DK_CUDA(cudaMallocAsync(&dl, sizeof(int64_t) * std::max<int64_t>(cap, 1), s));
    DK_CUDA(cudaMallocAsync(&dc, sizeof(unsigned long long), s));
    DK_CUDA(cudaMemsetAsync(dc, 0, sizeof(unsigned long long), s));
    const int64_t nchunk = (out_end + kRejChunk - 1) / kRejChunk;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((nchunk + 127) / 128, (int64_t)st().sm_count * 16));
    if (nchunk > 0) {
      k_pcg_rejects<<<blocks, 128, 0, s>>>(u128_of(state), u128_of(inc), out_end, dl, dc, cap);
      DK_CUDA(cudaGetLastError());
      st().launches++;
    }
    unsigned long long n = 0;
    DK_CUDA(cudaMemcpyAsync(&n, dc, sizeof n, cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    const int64_t k = std::min<int64_t>((int64_t)n, cap);
    std::vector<int64_t> h(k);
    if (k) DK_CUDA(cudaMemcpy(h.data(), dl, sizeof(int64_t) * k, cudaMemcpyDeviceToHost));
    std::sort(h.begin(), h.end());
    std::copy(h.begin(), h.end(), out);
    *count = (int64_t)n;
    DK_CUDA(cudaFreeAsync(dl, s));
    DK_CUDA(cudaFreeAsync(dc, s));
  });
}

int dk_pcg64_fill(int64_t sid, const int64_t* lo, const int64_t* hi, const uint64_t* state, const uint64_t* inc,
                  int kind, double scale, const int64_t* breaks, int64_t nbreaks) {
  return guard([&] {
    require_init();
    Store& so = store_of(sid);
    if (so.dtype != DK_F64) fail(DK_ERR_UNSUPPORTED, "pcg64 fill of a non-f64 store");
    if (so.rank < 1 || so.rank > 2) fail(DK_ERR_UNSUPPORTED, "pcg64 fill supports rank 1 and 2 stores");
    int64_t r0 = 0, r1 = 1, c0 = lo[so.rank - 1], c1 = hi[so.rank - 1], L = so.ext[so.rank - 1];
    if (so.rank == 2) r0 = lo[0], r1 = hi[0];
    if (r1 <= r0 || c1 <= c0) return;
    const int64_t first = r0 * L + c0, last = (r1 - 1) * L + c1;
    store_ensure_bytes(so, (size_t)first * 8, (size_t)last * 8);
    cudaStream_t s = st().stream;
    int64_t* db = nullptr;
    if (nbreaks > 0) {
      DK_CUDA(cudaMallocAsync(&db, sizeof(int64_t) * nbreaks, s));
      DK_CUDA(cudaMemcpyAsync(db, breaks, sizeof(int64_t) * nbreaks, cudaMemcpyHostToDevice, s));
    }
    const int64_t segs = (r1 - r0) * ((c1 - c0 + kSeg - 1) / kSeg);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((segs + 255) / 256, (int64_t)st().sm_count * 8));
    k_pcg_fill<<<blocks, 256, 0, s>>>((double*)so.base, L, r0, r1, c0, c1, u128_of(state), u128_of(inc), kind, scale,
                                      db, nbreaks);
    DK_CUDA(cudaGetLastError());
    st().launches++;
    if (db) {
      DK_CUDA(cudaStreamSynchronize(s));  // the host breaks buffer must outlive the copy
      DK_CUDA(cudaFreeAsync(db, s));
    }
  });
}

}  // extern "C"
