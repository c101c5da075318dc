// Inter-GPU movement for the partition -> GPU mapping (NCCL over NVLink 5 /
// NVSwitch).  The reference has no communication at all: its
// launch points share one host heap.  Here every rank holds only the
// sub-stores of its own points, so the three exchanges the fusion guarantee
// leaves between launches become:
//   * halo rows of aliased stencil views and replicated (NonePart) reads of
//     tile-written vectors   -> dk_comm_exchange (grouped ncclSend/ncclRecv
//     of store rects, packed only when a rect is not contiguous);
//   * per-point reduction partials -> dk_comm_allgather_f64, folded in launch
//     point order on every rank (executor.py:193-195 order, bit-reproducible).
// The transfer plan itself is computed identically on every rank by the
// host-side coherence planner (paper_2406_18109_b200/coherence.py).

#include <nccl.h>

#include <cstring>
#include <vector>

#include "dk_internal.h"

namespace dk {

#define DK_NCCL(x)                                                                                 \
  do {                                                                                             \
    ncclResult_t r_ = (x);                                                                         \
    if (r_ != ncclSuccess) fail(DK_ERR_NCCL, "%s: %s (%s:%d)", #x, ncclGetErrorString(r_), __FILE__, __LINE__); \
  } while (0)

static ncclComm_t comm() {
  if (!st().comm) fail(DK_ERR_STATE, "dk_comm_init has not been called");
  return (ncclComm_t)st().comm;
}

struct RectView {
  dk_view v;
  bool contiguous;
  int64_t first;  // element offset of the rect start
  int64_t count;
};

static RectView rect_view(Store& s, const int64_t* lo, const int64_t* hi) {
  RectView rv;
  memset(&rv.v, 0, sizeof rv.v);
  const int r = s.rank;
  int64_t str[4] = {1, 1, 1, 1};
  for (int d = r - 2; d >= 0; --d) str[d] = str[d + 1] * s.ext[d + 1];
  rv.first = 0;
  rv.count = 1;
  for (int d = 0; d < r; ++d) {
    int64_t l = std::max<int64_t>(0, lo[d]), h = std::min<int64_t>(s.ext[d], hi[d]);
    if (h < l) h = l;
    rv.v.ext[d] = h - l;
    rv.v.stride[d] = str[d];
    rv.first += l * str[d];
    rv.count *= (h - l);
  }
  rv.v.rank = r;
  rv.v.dtype = s.dtype;
  rv.v.ptr = (uint64_t)s.base + (uint64_t)rv.first * s.esize;
  // contiguous iff every dim after the first non-singleton one is full
  int d0 = 0;
  while (d0 < r && rv.v.ext[d0] == 1) ++d0;
  rv.contiguous = true;
  for (int d = d0 + 1; d < r; ++d)
    if (rv.v.ext[d] != s.ext[d]) rv.contiguous = false;
  return rv;
}

// Consume the flags of one board slot: thread (q, j) waits until point j of
// rank q has published (its kernel's last CTA wrote the totals and then the
// flag with release semantics at system scope), then clears the flag.  A
// peer that never publishes is a protocol bug: trap after 10 s instead of
// hanging the GPU.
struct P2PCounts {
  int c[kP2PWMax];
};

struct P2PFolds {
  int n;
  uint64_t target[DK_P2P_FOLDS];
  int64_t first[DK_P2P_FOLDS], stride[DK_P2P_FOLDS];
  int32_t cnt[DK_P2P_FOLDS];
};

__global__ void k_p2p_wait(unsigned int* flags, P2PCounts counts, int world, unsigned tag);

// wait for the slot's flags, then fold in the given order (one thread: the
// order of the adds is the reference's point order, executor.py:193-195)
__global__ void k_p2p_wait_fold(unsigned int* flags, P2PCounts counts, int world, unsigned tag, const double* g,
                                P2PFolds f) {
  const int q = threadIdx.x / DK_P2P_POINTS, j = threadIdx.x % DK_P2P_POINTS;
  if (q < world && j < counts.c[q]) {
    unsigned int* fl = flags + q * DK_P2P_POINTS + j;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
      if (v == tag) break;
      if (v != 0u) {
        printf("dk_p2p_wait_fold: rank %d point %d flag holds tag %u, expected %u\n", q, j, v, tag);
        __trap();
      }
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) __trap();
      __nanosleep(64);
    }
    *fl = 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int i = 0; i < f.n; ++i) {
      double* tp = (double*)f.target[i];
      double a = *tp;
      for (int k = 0; k < f.cnt[i]; ++k) a = __dadd_rn(a, g[f.first[i] + k * f.stride[i]]);
      *tp = a;
    }
  }
}

__global__ void k_p2p_wait(unsigned int* flags, P2PCounts counts, int world, unsigned tag) {
  const int q = threadIdx.x / DK_P2P_POINTS, j = threadIdx.x % DK_P2P_POINTS;
  if (q < world && j < counts.c[q]) {
    unsigned int* f = flags + q * DK_P2P_POINTS + j;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (v == tag) break;
      if (v != 0u) {
        // another epoch's publish in this slot: the ring invariant is broken
        printf("dk_p2p_wait: rank %d point %d flag holds tag %u, expected %u\n", q, j, v, tag);
        __trap();
      }
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) __trap();
      __nanosleep(64);
    }
    *f = 0u;
  }
  __threadfence_system();
}

// ---- halo moves over peer memory (dk_p2p_exchange) ----------------------------
// One CTA per (peer, direction).  A send CTA waits for the receiver's ack of
// the exchange two epochs back on this mailbox parity, copies its rects into
// the receiver's mailbox [me][parity] (peer stores over NVLink), then thread 0
// publishes the epoch's tag into the receiver's mail flag with release
// semantics at system scope.  A receive CTA waits for that tag (acquire),
// copies the mailbox into its store rects and acks into the sender's board.
// Flags and acks hold the tag of the latest message (never cleared: the
// next value a parity sees is two messages on); 10 s without progress traps
// (never a hang).
constexpr int kXMaxItems = 8;
struct XItem {
  dk_view v;     // store rect (8- or 4-byte elements)
  int64_t off;   // byte offset inside the mailbox
  int64_t count; // elements
};
struct XCta {
  int dir;            // 0 send, 1 recv
  int nitems;
  unsigned tag, prev; // this epoch's tag; the ack to wait for before sending (0: none)
  uint64_t mail;      // send: receiver's mailbox base; recv: my mailbox base
  uint64_t flag;      // send: receiver's mail flag; recv: my mail flag
  uint64_t ack;       // send: my ack flag (written by the receiver); recv: the sender's ack flag
  XItem item[kXMaxItems];
};
struct XArgs {
  int ncta;
  XCta cta[2 * kP2PWMax];
};
static_assert(sizeof(XArgs) < 32000, "kernel parameter block");

__device__ __forceinline__ void x_wait(const unsigned int* f, unsigned tag, const char* what, int cta) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (v == tag) return;  // flags hold the latest message's tag (never cleared)
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 10000000000ull) {
      printf("dk_p2p_exchange: cta %d timed out waiting for %s tag %u (last %u)\n", cta, what, tag, v);
      __trap();
    }
    __nanosleep(32);
  }
}

__device__ __forceinline__ int64_t x_elem_off(const dk_view& v, int64_t i) {
  int64_t o = 0;
  for (int d = v.rank - 1; d >= 0; --d) {
    const int64_t e = v.ext[d];
    o += (i % e) * v.stride[d];
    i /= e;
  }
  return o;
}

// one CTA moves one rect between a store view and its dense mailbox image:
// contiguous rects as 16-byte vectors when both ends allow it, else row by row
// (rank <= 2 views: rows are contiguous runs of ext[rank-1] elements)
__device__ __forceinline__ void x_copy(const XItem& it, char* dst, const char* src, bool pack) {
  const int es = it.v.dtype == DK_F64 ? 8 : 4;
  const int r = it.v.rank;
  const int64_t inner = r ? it.v.ext[r - 1] : 1;
  const bool contiguous = r <= 1 || it.v.stride[r - 2] == inner || it.count == inner;
  if (contiguous) {
    const int64_t bytes = it.count * es;
    if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
      const int64_t nv = bytes / 16;
      for (int64_t i = threadIdx.x; i < nv; i += blockDim.x)
        ((int4*)dst)[i] = ((const int4*)src)[i];
      for (int64_t b = nv * 16 + threadIdx.x * 4; b < bytes; b += blockDim.x * 4)
        *(int*)(dst + b) = *(const int*)(src + b);
    } else if (es == 8) {
      for (int64_t i = threadIdx.x; i < it.count; i += blockDim.x) ((double*)dst)[i] = ((const double*)src)[i];
    } else {
      for (int64_t i = threadIdx.x; i < it.count; i += blockDim.x) ((int*)dst)[i] = ((const int*)src)[i];
    }
    return;
  }
  if (r == 2) {
    const int64_t rows = it.v.ext[0], rs = it.v.stride[0];
    for (int64_t row = 0; row < rows; ++row)
      for (int64_t j = threadIdx.x; j < inner; j += blockDim.x) {
        const int64_t m = row * inner + j, o = row * rs + j;
        if (es == 8) {
          if (pack) ((double*)dst)[m] = ((const double*)src)[o];
          else ((double*)dst)[o] = ((const double*)src)[m];
        } else {
          if (pack) ((int*)dst)[m] = ((const int*)src)[o];
          else ((int*)dst)[o] = ((const int*)src)[m];
        }
      }
    return;
  }
  for (int64_t i = threadIdx.x; i < it.count; i += blockDim.x) {
    const int64_t o = x_elem_off(it.v, i);
    if (es == 8) {
      if (pack) ((double*)dst)[i] = ((const double*)src)[o];
      else ((double*)dst)[o] = ((const double*)src)[i];
    } else {
      if (pack) ((int*)dst)[i] = ((const int*)src)[o];
      else ((int*)dst)[o] = ((const int*)src)[i];
    }
  }
}

__global__ void __launch_bounds__(1024) k_p2p_xchg(XArgs a) {
  const XCta& c = a.cta[blockIdx.x];
  if (c.dir == 0) {
    if (c.prev && threadIdx.x == 0) x_wait((const unsigned int*)c.ack, c.prev, "ack", blockIdx.x);
    __syncthreads();
    for (int k = 0; k < c.nitems; ++k) {
      const XItem& it = c.item[k];
      x_copy(it, (char*)c.mail + it.off, (const char*)it.v.ptr, true);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(c.flag), "r"(c.tag) : "memory");
    }
  } else {
    if (threadIdx.x == 0) x_wait((const unsigned int*)c.flag, c.tag, "mail", blockIdx.x);
    __syncthreads();
    for (int k = 0; k < c.nitems; ++k) {
      const XItem& it = c.item[k];
      x_copy(it, (char*)it.v.ptr, (const char*)c.mail + it.off, false);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(c.ack), "r"(c.tag) : "memory");
  }
}

}  // namespace dk

using namespace dk;

extern "C" {

int dk_p2p_exchange(int n, const int64_t* sids, const int32_t* peers, const int32_t* dirs, const int64_t* los,
                    const int64_t* his) {
  return guard([&] {
    require_init();
    require_not_capturing("dk_p2p_exchange");
    State& S = st();
    if (!S.p2p) fail(DK_ERR_STATE, "dk_p2p_init has not enabled peer memory");
    if (n <= 0) return;
    NvtxRange nv("dk_p2p_exchange", n);
    XArgs a = {};
    int cta_of[2][kP2PWMax];
    for (auto& r : cta_of)
      for (int& x : r) x = -1;
    for (int i = 0; i < n; ++i) {
      const int q = peers[i], dir = dirs[i];
      if (q < 0 || q >= S.world || q == S.rank) fail(DK_ERR_ARG, "bad peer %d", q);
      Store& so = store_of(sids[i]);
      RectView rv = rect_view(so, los + 4 * i, his + 4 * i);
      if (rv.count == 0) continue;
      int64_t last = rv.first;
      for (int d = 0; d < so.rank; ++d) last += (rv.v.ext[d] - 1) * rv.v.stride[d];
      store_ensure_bytes(so, (size_t)rv.first * so.esize, (size_t)(last + 1) * so.esize);
      rv.v.ptr = (uint64_t)so.base + (uint64_t)rv.first * so.esize;
      int& ci = cta_of[dir][q];
      if (ci < 0) {
        ci = a.ncta++;
        XCta& c = a.cta[ci];
        const int64_t e = dir == 0 ? S.xsend[q] : S.xrecv[q];
        const int par = (int)(e & 1);
        c.dir = dir;
        c.tag = p2p_tag(e);
        c.prev = e >= 2 ? p2p_tag(e - 2) : 0u;
        if (dir == 0) {
          c.mail = S.peer_board[q] + mail_data_off(S.rank, par);
          c.flag = S.peer_board[q] + mail_flag_off(S.rank, par);
          c.ack = (uint64_t)S.board + mail_ack_off(q, par);
        } else {
          c.mail = (uint64_t)S.board + mail_data_off(q, par);
          c.flag = (uint64_t)S.board + mail_flag_off(q, par);
          c.ack = S.peer_board[q] + mail_ack_off(S.rank, par);
        }
      }
      XCta& c = a.cta[ci];
      if (c.nitems >= kXMaxItems) fail(DK_ERR_UNSUPPORTED, "more than %d rects for one peer", kXMaxItems);
      int64_t off = 0;
      if (c.nitems) {
        const XItem& pv = c.item[c.nitems - 1];
        off = pv.off + ((pv.count * (pv.v.dtype == DK_F64 ? 8 : 4) + 15) & ~(int64_t)15);
      }
      if (off + rv.count * (int64_t)so.esize > (int64_t)kMailSlot)
        fail(DK_ERR_UNSUPPORTED, "halo to rank %d exceeds the %d-byte mailbox", q, (int)kMailSlot);
      XItem& it = c.item[c.nitems++];
      it.v = rv.v;
      it.off = off;
      it.count = rv.count;
    }
    if (a.ncta == 0) return;
    k_p2p_xchg<<<a.ncta, 1024, 0, S.stream>>>(a);
    DK_CUDA(cudaGetLastError());
    S.launches++;
    for (int q = 0; q < S.world; ++q) {
      if (cta_of[0][q] >= 0) S.xsend[q]++;
      if (cta_of[1][q] >= 0) S.xrecv[q]++;
    }
  });
}

static void dma_move(int n, const int64_t* sids, const int32_t* peers, const int64_t* los, const int64_t* his,
                     bool send) {
  require_init();
  require_not_capturing(send ? "dk_dma_send" : "dk_dma_recv");
  State& S = st();
  if (!S.p2p) fail(DK_ERR_STATE, "dk_p2p_init has not enabled peer memory");
  CUstream cs = (CUstream)S.stream;
  // group the rects by peer, in order (both ends see the same order: the plan is replicated)
  for (int q = 0; q < S.world; ++q) {
    int64_t off = 0;
    bool any = false;
    const int64_t k = send ? S.xsend[q] : S.xrecv[q];
    const int par = (int)(k & 1);
    const unsigned tag = p2p_tag(k);
    for (int i = 0; i < n; ++i) {
      if (peers[i] != q) continue;
      if (q == S.rank || q < 0 || q >= S.world) fail(DK_ERR_ARG, "bad peer %d", q);
      Store& so = store_of(sids[i]);
      RectView rv = rect_view(so, los + 4 * i, his + 4 * i);
      if (rv.count == 0) continue;
      if (!rv.contiguous) fail(DK_ERR_UNSUPPORTED, "dk_dma_*: rect of store %lld is not contiguous", (long long)sids[i]);
      store_ensure_bytes(so, (size_t)rv.first * so.esize, (size_t)(rv.first + rv.count) * so.esize);
      const size_t bytes = (size_t)rv.count * so.esize;
      if (off + (int64_t)bytes > (int64_t)kMailSlot) fail(DK_ERR_UNSUPPORTED, "halo exceeds the mailbox");
      void* store_ptr = (void*)((uint64_t)so.base + (uint64_t)rv.first * so.esize);
      if (!any) {
        any = true;
        if (send && k >= 2)  // the receiver consumed the message two before on this parity
          DK_CU(cuStreamWaitValue32(cs, (CUdeviceptr)((uint64_t)S.board + mail_ack_off(q, par)), p2p_tag(k - 2),
                                    CU_STREAM_WAIT_VALUE_GEQ));
        if (!send)
          DK_CU(cuStreamWaitValue32(cs, (CUdeviceptr)((uint64_t)S.board + mail_flag_off(q, par)), tag,
                                    CU_STREAM_WAIT_VALUE_EQ));
      }
      if (send)
        DK_CUDA(cudaMemcpyAsync((void*)(S.peer_board[q] + mail_data_off(S.rank, par) + off), store_ptr, bytes,
                                cudaMemcpyDeviceToDevice, S.stream));
      else
        DK_CUDA(cudaMemcpyAsync(store_ptr, (void*)((uint64_t)S.board + mail_data_off(q, par) + off), bytes,
                                cudaMemcpyDeviceToDevice, S.stream));
      off += (int64_t)((bytes + 15) & ~(size_t)15);
    }
    if (!any) continue;
    if (send) {
      DK_CU(cuStreamWriteValue32(cs, (CUdeviceptr)(S.peer_board[q] + mail_flag_off(S.rank, par)), tag,
                                 CU_STREAM_WRITE_VALUE_DEFAULT));
      S.xsend[q]++;
    } else {
      DK_CU(cuStreamWriteValue32(cs, (CUdeviceptr)(S.peer_board[q] + mail_ack_off(S.rank, par)), tag,
                                 CU_STREAM_WRITE_VALUE_DEFAULT));
      S.xrecv[q]++;
    }
  }
}

int dk_dma_send(int n, const int64_t* sids, const int32_t* peers, const int64_t* los, const int64_t* his) {
  return guard([&] {
    NvtxRange nv("dk_dma_send", n);
    dma_move(n, sids, peers, los, his, true);
  });
}

int dk_dma_recv(int n, const int64_t* sids, const int32_t* peers, const int64_t* los, const int64_t* his) {
  return guard([&] {
    NvtxRange nv("dk_dma_recv", n);
    dma_move(n, sids, peers, los, his, false);
  });
}

int dk_comm_unique_id(uint8_t* out128) {
  return guard([&] {
    ncclUniqueId id;
    DK_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "nccl id size");
    memcpy(out128, &id, 128);
  });
}

int dk_comm_init(int rank, int world, const uint8_t* id128) {
  return guard([&] {
    require_init();
    if (st().comm) {
      // one communicator per process; later executors of the same job reuse it
      if (st().rank == rank && st().world == world) return;
      fail(DK_ERR_STATE, "communicator already initialised for rank %d of %d", st().rank, st().world);
    }
    ncclUniqueId id;
    memcpy(&id, id128, 128);
    ncclComm_t c;
    DK_NCCL(ncclCommInitRank(&c, world, id, rank));
    st().comm = c;
    st().rank = rank;
    st().world = world;
  });
}

int dk_comm_destroy(void) {
  return guard([&] {
    if (!st().comm) return;
    State& S = st();
    if (S.p2p) {
      cudaDeviceSynchronize();
      for (int q = 0; q < S.world; ++q)
        if (q != S.rank && S.peer_board[q]) cudaIpcCloseMemHandle((void*)S.peer_board[q]);
      cudaFree(S.board);
      S.board = nullptr;
      memset(S.peer_board, 0, sizeof S.peer_board);
      S.p2p = false;
    }
    ncclCommDestroy((ncclComm_t)st().comm);
    st().comm = nullptr;
  });
}

int dk_comm_exchange(int n, const int64_t* sids, const int32_t* peers, const int32_t* dirs, const int64_t* los,
                     const int64_t* his) {
  return guard([&] {
    require_init();
    if (n <= 0) return;
    NvtxRange nv("dk_comm_exchange", n);
    ncclComm_t c = comm();
    cudaStream_t s = st().stream;
    std::vector<RectView> rvs(n);
    std::vector<void*> staging(n, nullptr);
    for (int i = 0; i < n; ++i) {
      Store& so = store_of(sids[i]);
      rvs[i] = rect_view(so, los + 4 * i, his + 4 * i);
      if (rvs[i].count == 0) continue;
      // back the span this rect touches
      int64_t last = rvs[i].first;
      for (int d = 0; d < so.rank; ++d) last += (rvs[i].v.ext[d] - 1) * rvs[i].v.stride[d];
      store_ensure_bytes(so, (size_t)rvs[i].first * so.esize, (size_t)(last + 1) * so.esize);
      rvs[i].v.ptr = (uint64_t)so.base + (uint64_t)rvs[i].first * so.esize;
      if (!rvs[i].contiguous) {
        if (so.esize != 8) fail(DK_ERR_UNSUPPORTED, "non-contiguous transfer of a 4-byte store");
        DK_CUDA(cudaMallocAsync(&staging[i], (size_t)rvs[i].count * 8, s));
        if (dirs[i] == 0) launch_pack(rvs[i].v, (double*)staging[i], s, false);
      }
    }
    DK_NCCL(ncclGroupStart());
    for (int i = 0; i < n; ++i) {
      if (rvs[i].count == 0) continue;
      Store& so = store_of(sids[i]);
      void* buf = rvs[i].contiguous ? (void*)rvs[i].v.ptr : staging[i];
      size_t bytes = (size_t)rvs[i].count * so.esize;
      if (dirs[i] == 0)
        DK_NCCL(ncclSend(buf, bytes, ncclUint8, peers[i], c, s));
      else
        DK_NCCL(ncclRecv(buf, bytes, ncclUint8, peers[i], c, s));
    }
    DK_NCCL(ncclGroupEnd());
    for (int i = 0; i < n; ++i) {
      if (!staging[i]) continue;
      if (dirs[i] == 1) launch_pack(rvs[i].v, (double*)staging[i], s, true);
      DK_CUDA(cudaFreeAsync(staging[i], s));
    }
  });
}

int dk_comm_allgather_f64(uint64_t src, uint64_t dst, int64_t count) {
  return guard([&] {
    require_init();
    DK_NCCL(ncclAllGather((const void*)src, (void*)dst, (size_t)count, ncclDouble, comm(), st().stream));
  });
}

int dk_p2p_init(int* enabled) {
  return guard([&] {
    require_init();
    ncclComm_t c = comm();
    State& S = st();
    *enabled = 0;
    if (S.p2p) {
      *enabled = 1;
      return;
    }
    cudaStream_t s = S.stream;
    int ok = S.world <= kP2PWMax && !getenv("DK_NO_P2P");
    cudaIpcMemHandle_t mine;
    memset(&mine, 0, sizeof mine);
    if (ok) ok = cudaMalloc(&S.board, kP2PBoardBytes) == cudaSuccess;
    if (ok) ok = cudaMemsetAsync(S.board, 0, kP2PBoardBytes, s) == cudaSuccess;
    if (ok) ok = cudaIpcGetMemHandle(&mine, S.board) == cudaSuccess;
    cudaGetLastError();
    // all-gather the IPC handles (and the success bits) over NCCL
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    char* dev = nullptr;
    DK_CUDA(cudaMalloc(&dev, hb * (S.world + 1) + 8));
    DK_CUDA(cudaMemcpyAsync(dev + hb * S.world, &mine, hb, cudaMemcpyHostToDevice, s));
    DK_NCCL(ncclAllGather(dev + hb * S.world, dev, hb, ncclUint8, c, s));
    std::vector<cudaIpcMemHandle_t> all(S.world);
    DK_CUDA(cudaMemcpyAsync(all.data(), dev, hb * S.world, cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    std::vector<int> opened(S.world, 0);
    for (int q = 0; q < S.world && ok; ++q) {
      if (q == S.rank) {
        S.peer_board[q] = (uint64_t)S.board;
        continue;
      }
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      S.peer_board[q] = (uint64_t)p;
      opened[q] = 1;
    }
    // every rank must agree before anyone takes the peer-memory path
    int* flag = (int*)(dev + hb * S.world);
    DK_CUDA(cudaMemcpyAsync(flag, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
    DK_NCCL(ncclAllReduce(flag, flag, 1, ncclInt32, ncclMin, c, s));
    int all_ok = 0;
    DK_CUDA(cudaMemcpyAsync(&all_ok, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    DK_CUDA(cudaFree(dev));
    if (!all_ok) {
      for (int q = 0; q < S.world; ++q)
        if (opened[q]) cudaIpcCloseMemHandle((void*)S.peer_board[q]);
      if (S.board) cudaFree(S.board);
      S.board = nullptr;
      memset(S.peer_board, 0, sizeof S.peer_board);
      cudaGetLastError();
      return;
    }
    S.p2p = true;
    *enabled = 1;
  });
}

int dk_p2p_wait(int64_t epoch, const int32_t* counts, uint64_t* gathered) {
  return guard([&] {
    require_init();
    require_not_capturing("dk_p2p_wait");
    NvtxRange nv("dk_p2p_wait", epoch);
    State& S = st();
    if (!S.p2p) fail(DK_ERR_STATE, "dk_p2p_init has not enabled peer-memory reductions");
    if (epoch < 0) fail(DK_ERR_ARG, "negative reduction epoch");
    const int slot = (int)(epoch % DK_P2P_SLOTS);
    P2PCounts pc = {};
    for (int q = 0; q < S.world; ++q) {
      if (counts[q] < 0 || counts[q] > DK_P2P_POINTS) fail(DK_ERR_ARG, "rank %d publishes %d points", q, counts[q]);
      pc.c[q] = counts[q];
    }
    char* b = (char*)S.board;
    k_p2p_wait<<<1, kP2PWMax * DK_P2P_POINTS, 0, S.stream>>>((unsigned int*)(b + p2p_flag_off(slot)), pc, S.world,
                                                            p2p_tag(epoch));
    DK_CUDA(cudaGetLastError());
    S.launches++;
    *gathered = (uint64_t)(b + p2p_data_off(slot));
  });
}

int dk_p2p_wait_fold(int64_t epoch, const int32_t* counts, int nfold, const uint64_t* targets,
                     const int64_t* firsts, const int64_t* strides, const int32_t* ns) {
  return guard([&] {
    require_init();
    require_not_capturing("dk_p2p_wait_fold");
    NvtxRange nv("dk_p2p_wait_fold", epoch);
    State& S = st();
    if (!S.p2p) fail(DK_ERR_STATE, "dk_p2p_init has not enabled peer-memory reductions");
    if (epoch < 0) fail(DK_ERR_ARG, "negative reduction epoch");
    if (nfold < 0 || nfold > DK_P2P_FOLDS) fail(DK_ERR_ARG, "%d folds (max %d)", nfold, DK_P2P_FOLDS);
    const int slot = (int)(epoch % DK_P2P_SLOTS);
    P2PCounts pc = {};
    for (int q = 0; q < S.world; ++q) {
      if (counts[q] < 0 || counts[q] > DK_P2P_POINTS) fail(DK_ERR_ARG, "rank %d publishes %d points", q, counts[q]);
      pc.c[q] = counts[q];
    }
    P2PFolds f = {};
    f.n = nfold;
    for (int i = 0; i < nfold; ++i) {
      f.target[i] = targets[i];
      f.first[i] = firsts[i];
      f.stride[i] = strides[i];
      f.cnt[i] = ns[i];
    }
    char* b = (char*)S.board;
    k_p2p_wait_fold<<<1, kP2PWMax * DK_P2P_POINTS, 0, S.stream>>>((unsigned int*)(b + p2p_flag_off(slot)), pc,
                                                                 S.world, p2p_tag(epoch),
                                                                 (const double*)(b + p2p_data_off(slot)), f);
    DK_CUDA(cudaGetLastError());
    S.launches++;
  });
}

int dk_comm_barrier(void) {
  return guard([&] {
    require_init();
    void* p = nullptr;
    DK_CUDA(cudaMallocAsync(&p, 64, st().stream));
    DK_NCCL(ncclAllReduce(p, p, 1, ncclInt32, ncclSum, comm(), st().stream));
    DK_CUDA(cudaFreeAsync(p, st().stream));
    DK_CUDA(cudaStreamSynchronize(st().stream));
  });
}

}  // extern "C"
