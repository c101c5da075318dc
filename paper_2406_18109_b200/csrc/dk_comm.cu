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

}  // namespace dk

using namespace dk;

extern "C" {

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
    ncclCommDestroy((ncclComm_t)st().comm);
    st().comm = nullptr;
  });
}

int dk_comm_exchange(int n, const int64_t* sids, const int32_t* peers, const int32_t* dirs, const int64_t* los,
                     const int64_t* his) {
  return guard([&] {
    require_init();
    if (n <= 0) return;
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
