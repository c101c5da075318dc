// Device heap and process/GPU binding for the B200 backend.
//
// Replaces the reference Heap (diffusekit executor.py:40-79): a store id maps
// to one row-major array.  On the GPU a large store reserves virtual address
// space for its whole extent (cuMemAddressReserve) and is backed by HBM only
// where this rank's launch points touch it (dk_store_ensure ->
// cuMemCreate/cuMemMap).  Global element offsets therefore stay valid on every
// rank, which keeps sub-store views identical to the reference's
// (_region, executor.py:119-121) while a rank holds only its partition and
// halo.  Freed stores keep their mappings in a size-keyed pool so the
// unfused path's per-task temporaries do not pay cuMemCreate each time.
// Small stores (<= 1 MiB, e.g. rank-0 reduction targets) use the
// stream-ordered allocator.

#include <algorithm>
#include <cstring>

#include "dk_internal.h"

namespace dk {

static thread_local std::string g_err;
static State g_state;

State& st() { return g_state; }

void destroy_graphs();  // defined with the graph registry below

void set_last_error(const std::string& msg) { g_err = msg; }

void fail(int code, const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw Error(code, buf);
}

void require_init() {
  if (!g_state.inited) fail(DK_ERR_STATE, "dk_init has not been called");
}

void require_not_capturing(const char* what) {
  if (g_state.capture_launch0 >= 0)
    fail(DK_ERR_STATE, "%s is not allowed while a graph capture is open (it cannot be replayed)", what);
}

Store& store_of(int64_t sid) {
  auto it = g_state.stores.find(sid);
  if (it == g_state.stores.end()) fail(DK_ERR_STATE, "unknown store %lld", (long long)sid);
  return it->second;
}

static const size_t kSmallStore = 1u << 20;

static void map_range(Store& s, size_t off, size_t size) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = g_state.device;
  CUmemGenericAllocationHandle h;
  CUresult r = cuMemCreate(&h, size, &prop, 0);
  if (r == CUDA_ERROR_OUT_OF_MEMORY && g_state.pool_bytes) {
    // give pooled physical memory back and retry once
    DK_CUDA(cudaStreamSynchronize(g_state.stream));
    for (auto& kv : g_state.va_pool) {
      for (auto& m : kv.second.maps) {
        cuMemUnmap(kv.second.base + m.off, m.size);
        cuMemRelease(m.h);
      }
      cuMemAddressFree(kv.second.base, kv.second.va_size);
    }
    g_state.va_pool.clear();
    g_state.pool_bytes = 0;
    r = cuMemCreate(&h, size, &prop, 0);
  }
  DK_CU(r);
  DK_CU(cuMemMap(s.base + off, size, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = g_state.device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  DK_CU(cuMemSetAccess(s.base + off, size, &acc, 1));
  s.maps.push_back({off, size, h});
  std::sort(s.maps.begin(), s.maps.end(), [](const Mapping& a, const Mapping& b) { return a.off < b.off; });
}

void store_ensure_bytes(Store& s, size_t lo, size_t hi) {
  if (s.small || hi <= lo) return;
  const size_t g = g_state.gran;
  lo = (lo / g) * g;
  hi = std::min(((hi + g - 1) / g) * g, s.va_size);
  size_t cur = lo;
  std::vector<std::pair<size_t, size_t>> gaps;
  for (const Mapping& m : s.maps) {
    if (m.off + m.size <= cur) continue;
    if (m.off >= hi) break;
    if (m.off > cur) gaps.push_back({cur, m.off - cur});
    cur = std::max(cur, m.off + m.size);
    if (cur >= hi) break;
  }
  if (cur < hi) gaps.push_back({cur, hi - cur});
  for (auto& g2 : gaps) map_range(s, g2.first, g2.second);
}

static void release_large(Store& s) {
  for (auto& m : s.maps) {
    cuMemUnmap(s.base + m.off, m.size);
    cuMemRelease(m.h);
  }
  cuMemAddressFree(s.base, s.va_size);
  s.maps.clear();
}

}  // namespace dk

using namespace dk;

extern "C" {

const char* dk_last_error(void) { return dk::g_err.c_str(); }

int dk_version(void) { return 1; }

int dk_init(int device) {
  return guard([&] {
    State& S = st();
    if (S.inited) {
      if (S.device != device) fail(DK_ERR_STATE, "already bound to device %d", S.device);
      return;
    }
    DK_CU(cuInit(0));
    DK_CUDA(cudaSetDevice(device));
    DK_CUDA(cudaFree(0));  // create / retain the primary context
    DK_CU(cuDeviceGet(&S.cudev, device));
    DK_CUDA(cudaDeviceGetAttribute(&S.sm_count, cudaDevAttrMultiProcessorCount, device));
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    size_t gran = 0;
    DK_CU(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    S.gran = gran ? gran : (2u << 20);
    DK_CUDA(cudaStreamCreateWithFlags(&S.own_stream, cudaStreamNonBlocking));
    S.stream = S.own_stream;
    S.device = device;
    S.inited = true;
  });
}

int dk_shutdown(void) {
  return guard([&] {
    State& S = st();
    if (!S.inited) return;
    cudaStreamSynchronize(S.stream);
    for (auto& kv : S.stores) {
      if (kv.second.small)
        cudaFree((void*)kv.second.base);
      else
        release_large(kv.second);
    }
    S.stores.clear();
    for (auto& kv : S.va_pool) release_large(kv.second);
    S.va_pool.clear();
    S.pool_bytes = 0;
    cudaStreamDestroy(S.own_stream);
    S.own_stream = S.stream = nullptr;
    S.inited = false;
  });
}

int dk_set_stream(uint64_t stream) {
  return guard([&] {
    require_init();
    st().stream = stream ? (cudaStream_t)stream : st().own_stream;
  });
}

int dk_get_stream(uint64_t* stream) {
  return guard([&] {
    require_init();
    *stream = (uint64_t)st().stream;
  });
}

int dk_sync(void) {
  return guard([&] {
    require_init();
    DK_CUDA(cudaStreamSynchronize(st().stream));
  });
}

int dk_device_info(int* sm_count, int64_t* free_bytes, int64_t* total_bytes) {
  return guard([&] {
    require_init();
    size_t f = 0, t = 0;
    DK_CUDA(cudaMemGetInfo(&f, &t));
    *sm_count = st().sm_count;
    *free_bytes = (int64_t)f;
    *total_bytes = (int64_t)t;
  });
}

int dk_timestamp(uint64_t buf, int64_t idx) {
  return guard([&] {
    require_init();
    launch_timestamp(buf, idx, st().stream);
  });
}

int dk_launch_count(int64_t* count) {
  return guard([&] { *count = st().launches; });
}

int dk_store_create(int64_t sid, int rank, const int64_t* extents, int dtype) {
  return guard([&] {
    require_init();
    State& S = st();
    if (S.stores.count(sid)) fail(DK_ERR_ARG, "store %lld already exists", (long long)sid);
    if (rank < 0 || rank > 4) fail(DK_ERR_UNSUPPORTED, "store rank %d > 4", rank);
    if (dtype != DK_F64 && dtype != DK_I32) fail(DK_ERR_ARG, "bad dtype %d", dtype);
    Store s;
    s.sid = sid;
    s.rank = rank;
    s.dtype = dtype;
    s.esize = dtype == DK_F64 ? 8 : 4;
    s.nelem = 1;
    for (int d = 0; d < rank; ++d) {
      if (extents[d] < 0) fail(DK_ERR_ARG, "negative extent");
      s.ext[d] = extents[d];
      s.nelem *= extents[d];
    }
    s.bytes = (size_t)s.nelem * s.esize;
    if (s.bytes <= kSmallStore) {
      s.small = true;
      void* p = nullptr;
      DK_CUDA(cudaMallocAsync(&p, std::max<size_t>(s.bytes, 16), S.stream));
      s.base = (CUdeviceptr)p;
    } else {
      s.va_size = ((s.bytes + S.gran - 1) / S.gran) * S.gran;
      auto it = S.va_pool.find(s.va_size);
      if (it != S.va_pool.end()) {
        s.base = it->second.base;
        s.maps = std::move(it->second.maps);
        for (auto& m : s.maps) S.pool_bytes -= m.size;
        S.va_pool.erase(it);
      } else {
        DK_CU(cuMemAddressReserve(&s.base, s.va_size, 0, 0, 0));
      }
    }
    S.stores.emplace(sid, std::move(s));
  });
}

int dk_store_ensure(int64_t sid, int64_t lo, int64_t hi) {
  return guard([&] {
    require_init();
    Store& s = store_of(sid);
    lo = std::max<int64_t>(lo, 0);
    hi = std::min<int64_t>(hi, s.nelem);
    if (hi > lo) store_ensure_bytes(s, (size_t)lo * s.esize, (size_t)hi * s.esize);
  });
}

int dk_store_free(int64_t sid) {
  return guard([&] {
    require_init();
    State& S = st();
    auto it = S.stores.find(sid);
    if (it == S.stores.end()) return;
    Store s = std::move(it->second);
    S.stores.erase(it);
    if (s.small) {
      DK_CUDA(cudaFreeAsync((void*)s.base, S.stream));
      return;
    }
    // keep VA + backing for reuse by a later store of the same size (stream
    // order makes the reuse safe); bound the pool so it cannot hoard HBM
    size_t mapped = 0;
    for (auto& m : s.maps) mapped += m.size;
    static const size_t kPoolCap = [] {
      const char* e = getenv("DK_VA_POOL_GB");  // 0 disables the pool
      return (size_t)(e ? atoll(e) : 64) << 30;
    }();
    if (S.pool_bytes + mapped > kPoolCap) {
      DK_CUDA(cudaStreamSynchronize(S.stream));
      release_large(s);
      return;
    }
    S.pool_bytes += mapped;
    Store pooled;
    pooled.base = s.base;
    pooled.va_size = s.va_size;
    pooled.maps = std::move(s.maps);
    S.va_pool.emplace(pooled.va_size, std::move(pooled));
  });
}

int dk_store_ptr(int64_t sid, uint64_t* dptr) {
  return guard([&] {
    require_init();
    *dptr = (uint64_t)store_of(sid).base;
  });
}

int dk_store_bytes_mapped(int64_t sid, int64_t* bytes) {
  return guard([&] {
    require_init();
    Store& s = store_of(sid);
    if (s.small) {
      *bytes = (int64_t)s.bytes;
      return;
    }
    size_t m = 0;
    for (auto& x : s.maps) m += x.size;
    *bytes = (int64_t)m;
  });
}

}  // extern "C"

namespace dk {

// Copy the rect [lo, hi) of a store to/from a host array shaped like the whole store.
static void rect_copy(int64_t sid, const int64_t* lo, const int64_t* hi, void* host, bool up) {
  require_init();
  require_not_capturing(up ? "dk_store_upload_rect" : "dk_store_download_rect");
  State& S = st();
  Store& s = store_of(sid);
  const int r = s.rank;
  int64_t e[4], l[4], h[4];
  for (int d = 0; d < r; ++d) {
    l[d] = std::max<int64_t>(0, lo[d]);
    h[d] = std::min<int64_t>(s.ext[d], hi[d]);
    if (h[d] <= l[d]) return;  // empty rect
    e[d] = s.ext[d];
  }
  char* hb = (char*)host;
  char* db = (char*)s.base;
  const size_t es = s.esize;
  if (r == 0) {
    store_ensure_bytes(s, 0, es);
    if (up)
      DK_CUDA(cudaMemcpyAsync(db, hb, es, cudaMemcpyHostToDevice, S.stream));
    else
      DK_CUDA(cudaMemcpyAsync(hb, db, es, cudaMemcpyDeviceToHost, S.stream));
    return;
  }
  // element strides of the full store
  int64_t str[4];
  str[r - 1] = 1;
  for (int d = r - 2; d >= 0; --d) str[d] = str[d + 1] * e[d + 1];
  // back the span the rect touches
  int64_t first = 0, last = 0;
  for (int d = 0; d < r; ++d) {
    first += l[d] * str[d];
    last += (h[d] - 1) * str[d];
  }
  store_ensure_bytes(s, (size_t)first * es, (size_t)(last + 1) * es);
  // merge trailing full dims into one contiguous run
  int inner = r - 1;
  int64_t run = h[inner] - l[inner];
  while (inner > 0 && l[inner] == 0 && h[inner] == e[inner]) {
    --inner;
    run = (h[inner] - l[inner]) * str[inner];
  }
  // rows over dim (inner-1) as a 2-D copy, loop over the rest
  const int rowdim = inner - 1;
  int64_t nrows = rowdim >= 0 ? h[rowdim] - l[rowdim] : 1;
  const size_t pitch = rowdim >= 0 ? (size_t)str[rowdim] * es : 0;
  int64_t outer_n = 1;
  for (int d = 0; d < rowdim; ++d) outer_n *= (h[d] - l[d]);
  for (int64_t o = 0; o < outer_n; ++o) {
    int64_t rem = o, off = 0;
    for (int d = rowdim - 1; d >= 0; --d) {
      int64_t n = h[d] - l[d];
      off += (l[d] + rem % n) * str[d];
      rem /= n;
    }
    if (rowdim >= 0) off += l[rowdim] * str[rowdim];
    off += l[inner] * str[inner];
    char* hp = hb + off * es;
    char* dp = db + off * es;
    const size_t w = (size_t)run * es;
    if (nrows == 1) {
      if (up)
        DK_CUDA(cudaMemcpyAsync(dp, hp, w, cudaMemcpyHostToDevice, S.stream));
      else
        DK_CUDA(cudaMemcpyAsync(hp, dp, w, cudaMemcpyDeviceToHost, S.stream));
    } else {
      if (up)
        DK_CUDA(cudaMemcpy2DAsync(dp, pitch, hp, pitch, w, nrows, cudaMemcpyHostToDevice, S.stream));
      else
        DK_CUDA(cudaMemcpy2DAsync(hp, pitch, dp, pitch, w, nrows, cudaMemcpyDeviceToHost, S.stream));
    }
  }
  if (!up) DK_CUDA(cudaStreamSynchronize(S.stream));
}

}  // namespace dk

extern "C" {

int dk_store_upload_rect(int64_t sid, const int64_t* lo, const int64_t* hi, const void* host) {
  return guard([&] { rect_copy(sid, lo, hi, const_cast<void*>(host), true); });
}

int dk_store_download_rect(int64_t sid, const int64_t* lo, const int64_t* hi, void* host) {
  return guard([&] { rect_copy(sid, lo, hi, host, false); });
}

int dk_store_fill(int64_t sid, int64_t lo, int64_t hi, double value) {
  return guard([&] {
    require_init();
    Store& s = store_of(sid);
    if (s.dtype != DK_F64) fail(DK_ERR_UNSUPPORTED, "fill of non-f64 store");
    lo = std::max<int64_t>(lo, 0);
    hi = std::min<int64_t>(hi, s.nelem);
    if (hi <= lo) return;
    store_ensure_bytes(s, (size_t)lo * 8, (size_t)hi * 8);
    launch_fill((double*)s.base + lo, hi - lo, value, st().stream);
  });
}

int dk_scratch_alloc(int64_t bytes, uint64_t* dptr) {
  return guard([&] {
    require_init();
    void* p = nullptr;
    DK_CUDA(cudaMallocAsync(&p, std::max<int64_t>(bytes, 16), st().stream));
    *dptr = (uint64_t)p;
  });
}

int dk_scratch_free(uint64_t dptr) {
  return guard([&] {
    require_init();
    if (dptr) DK_CUDA(cudaFreeAsync((void*)dptr, st().stream));
  });
}

int dk_memset_zero(uint64_t dptr, int64_t bytes) {
  return guard([&] {
    require_init();
    if (bytes > 0) DK_CUDA(cudaMemsetAsync((void*)dptr, 0, bytes, st().stream));
  });
}

int dk_memcpy_d2h(void* host, uint64_t dptr, int64_t bytes) {
  return guard([&] {
    require_init();
    DK_CUDA(cudaMemcpyAsync(host, (void*)dptr, bytes, cudaMemcpyDeviceToHost, st().stream));
    DK_CUDA(cudaStreamSynchronize(st().stream));
  });
}

int dk_memcpy_h2d(uint64_t dptr, const void* host, int64_t bytes) {
  return guard([&] {
    require_init();
    DK_CUDA(cudaMemcpyAsync((void*)dptr, host, bytes, cudaMemcpyHostToDevice, st().stream));
  });
}

int dk_memcpy_d2h_async(void* host, uint64_t dptr, int64_t bytes) {
  return guard([&] {
    require_init();
    DK_CUDA(cudaMemcpyAsync(host, (void*)dptr, bytes, cudaMemcpyDeviceToHost, st().stream));
  });
}

int dk_stream_new(uint64_t* stream) {
  return guard([&] {
    require_init();
    cudaStream_t s;
    DK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream = (uint64_t)s;
  });
}

int dk_event_new(uint64_t* event) {
  return guard([&] {
    require_init();
    cudaEvent_t e;
    DK_CUDA(cudaEventCreate(&e));
    *event = (uint64_t)e;
  });
}

int dk_event_record(uint64_t event) {
  return guard([&] { DK_CUDA(cudaEventRecord((cudaEvent_t)event, st().stream)); });
}

int dk_stream_wait_event(uint64_t event) {
  return guard([&] { DK_CUDA(cudaStreamWaitEvent(st().stream, (cudaEvent_t)event, 0)); });
}

int dk_event_sync(uint64_t event) {
  return guard([&] { DK_CUDA(cudaEventSynchronize((cudaEvent_t)event)); });
}

int dk_event_elapsed_ms(uint64_t start, uint64_t stop, float* ms) {
  return guard([&] { DK_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop)); });
}

int dk_host_alloc(int64_t bytes, void** host) {
  return guard([&] {
    require_init();
    DK_CUDA(cudaHostAlloc(host, std::max<int64_t>(bytes, 16), cudaHostAllocDefault));
  });
}

int dk_host_free(void* host) {
  return guard([&] {
    if (host) DK_CUDA(cudaFreeHost(host));
  });
}

int dk_accum(const dk_view* target, uint64_t vals, int64_t first, int64_t stride, int nvals) {
  return guard([&] {
    require_init();
    if (target->dtype != DK_F64) fail(DK_ERR_UNSUPPORTED, "accumulate into non-f64 view");
    if (nvals <= 0) return;
    launch_accum(*target, (const double*)vals + first, stride, nvals, st().stream);
  });
}

int dk_builtin(const char* kind, const dk_view* views, int nviews, const int32_t* writes) {
  return guard([&] {
    require_init();
    NvtxRange nv(kind, st().launches);
    launch_builtin(kind, views, nviews, writes, st().stream);
  });
}

int dk_spmv_csr_dot(const dk_view* views, uint64_t parts, int64_t x_row0, int* nparts) {
  return guard([&] {
    require_init();
    NvtxRange nv("SPMV_CSR+dot", st().launches);
    *nparts = launch_spmv_csr_dot(views, (double*)parts, x_row0, st().stream);
  });
}

}  // extern "C"

// ---- CUDA graphs of memo-hit windows --------------------------
// A replayed iteration whose launches are already in the prepared-launch cache
// is captured once from the library stream and relaunched as one graph: the
// device work is identical (same kernels, bindings and transfers), the host
// pays one cudaGraphLaunch instead of the front end's per-window dispatch.

namespace {
struct GraphRec {
  cudaGraphExec_t exec;
  int64_t kernels;
};
std::unordered_map<uint64_t, GraphRec> g_graphs;
uint64_t g_next_graph = 1;
}  // namespace

namespace dk {
void destroy_graphs() {
  for (auto& kv : g_graphs) cudaGraphExecDestroy(kv.second.exec);
  g_graphs.clear();
}
}  // namespace dk

extern "C" {

int dk_graph_begin(void) {
  return guard([&] {
    require_init();
    if (st().capture_launch0 >= 0) fail(DK_ERR_ARG, "a graph capture is already open");
    DK_CUDA(cudaStreamBeginCapture(st().stream, cudaStreamCaptureModeRelaxed));
    st().capture_launch0 = st().launches;
  });
}

int dk_graph_end(uint64_t* graph) {
  return guard([&] {
    require_init();
    if (st().capture_launch0 < 0) fail(DK_ERR_ARG, "no graph capture is open");
    const int64_t k = st().launches - st().capture_launch0;
    st().capture_launch0 = -1;
    st().launches -= k;  // captured, not launched
    cudaGraph_t g = nullptr;
    DK_CUDA(cudaStreamEndCapture(st().stream, &g));
    cudaGraphExec_t e = nullptr;
    cudaError_t r = cudaGraphInstantiate(&e, g, 0);
    cudaGraphDestroy(g);
    DK_CUDA(r);
    const uint64_t id = g_next_graph++;
    g_graphs[id] = GraphRec{e, k};
    *graph = id;
  });
}

int dk_graph_launch(uint64_t graph) {
  return guard([&] {
    require_init();
    auto it = g_graphs.find(graph);
    if (it == g_graphs.end()) fail(DK_ERR_ARG, "unknown graph %llu", (unsigned long long)graph);
    DK_CUDA(cudaGraphLaunch(it->second.exec, st().stream));
    st().launches += it->second.kernels;
  });
}

int dk_graph_destroy(uint64_t graph) {
  return guard([&] {
    auto it = g_graphs.find(graph);
    if (it == g_graphs.end()) fail(DK_ERR_ARG, "unknown graph %llu", (unsigned long long)graph);
    DK_CUDA(cudaGraphExecDestroy(it->second.exec));
    g_graphs.erase(it);
  });
}

}  // extern "C"
