// Internal state shared by the runtime translation units (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/dk_b200.h"

namespace dk {

// NVTX range around each C-ABI launch entry point (named by kind, payload = kernel
// handle or launch count): visible to Nsight tools, a no-op without one attached.
struct NvtxRange {
  NvtxRange(const char* name, int64_t payload) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    a.payloadType = NVTX_PAYLOAD_TYPE_INT64;
    a.payload.llValue = payload;
    nvtxRangePushEx(&a);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const char* fmt, ...);
void set_last_error(const std::string& msg);

#define DK_CUDA(x)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      ::dk::fail(e_ == cudaErrorMemoryAllocation ? DK_ERR_OOM : DK_ERR_CUDA, "%s: %s (%s:%d)", \
                 #x, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
  } while (0)

#define DK_CU(x)                                                                   \
  do {                                                                             \
    CUresult r_ = (x);                                                             \
    if (r_ != CUDA_SUCCESS) {                                                      \
      const char* s_ = nullptr;                                                    \
      cuGetErrorString(r_, &s_);                                                   \
      ::dk::fail(r_ == CUDA_ERROR_OUT_OF_MEMORY ? DK_ERR_OOM : DK_ERR_CUDA,        \
                 "%s: %s (%s:%d)", #x, s_ ? s_ : "?", __FILE__, __LINE__);         \
    }                                                                              \
  } while (0)

// C-ABI wrapper: run the body, convert exceptions into status codes.
template <class F>
int guard(F&& f) {
  try {
    f();
    return DK_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return DK_ERR_STATE;
  }
}

struct Mapping {
  size_t off, size;
  CUmemGenericAllocationHandle h;
};

struct Store {
  int64_t sid = -1;
  int rank = 0;
  int64_t ext[4] = {1, 1, 1, 1};
  int dtype = DK_F64;
  size_t esize = 8;
  int64_t nelem = 1;
  size_t bytes = 0;
  bool small = false;
  CUdeviceptr base = 0;  // small: cudaMallocAsync; large: reserved VA
  size_t va_size = 0;
  std::vector<Mapping> maps;  // sorted by off, disjoint (large stores)
};

struct State {
  bool inited = false;
  int device = -1;
  CUdevice cudev = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  size_t gran = 2u << 20;
  std::unordered_map<int64_t, Store> stores;
  std::multimap<size_t, Store> va_pool;  // freed large stores kept mapped, by va_size
  size_t pool_bytes = 0;
  int64_t launches = 0;
  // >= 0 while a CUDA-graph capture is open on `stream` (launch count at dk_graph_begin)
  int64_t capture_launch0 = -1;
  // collectives
  void* comm = nullptr;
  int rank = 0, world = 1;
  // peer-memory reduction boards (dk_p2p_init): own board + every rank's mapping
  bool p2p = false;
  void* board = nullptr;
  uint64_t peer_board[8] = {};
  // halo mailbox messages sent to / received from each peer so far (dk_p2p_exchange)
  int64_t xsend[8] = {}, xrecv[8] = {};
};

// board layout: [slot][kP2PWMax][DK_P2P_POINTS][DK_P2P_RED] doubles, then
// [slot][kP2PWMax][DK_P2P_POINTS] u32 flags
constexpr int kP2PWMax = 8;
constexpr size_t kP2PSlotBytes = (size_t)kP2PWMax * DK_P2P_POINTS * DK_P2P_RED * 8;
constexpr size_t kP2PFlagBytes = (size_t)kP2PWMax * DK_P2P_POINTS * 4;
inline size_t p2p_data_off(int slot) { return (size_t)slot * kP2PSlotBytes; }
inline size_t p2p_flag_off(int slot) { return DK_P2P_SLOTS * kP2PSlotBytes + (size_t)slot * kP2PFlagBytes; }
constexpr size_t kP2PRedBytes = DK_P2P_SLOTS * (kP2PSlotBytes + kP2PFlagBytes);
// halo mailboxes after the reduction ring: data [src rank][parity], then mail
// flags [src rank][parity] (raised by the sender), then ack flags [dst rank][parity]
// (raised by the receiver in the sender's board)
constexpr size_t kMailSlot = DK_P2P_MAIL_BYTES;
inline size_t mail_data_off(int src, int par) { return kP2PRedBytes + (size_t)(src * 2 + par) * kMailSlot; }
inline size_t mail_flag_off(int src, int par) {
  return kP2PRedBytes + (size_t)kP2PWMax * 2 * kMailSlot + (size_t)(src * 2 + par) * 4;
}
inline size_t mail_ack_off(int dst, int par) {
  return kP2PRedBytes + (size_t)kP2PWMax * 2 * kMailSlot + 256 + (size_t)(dst * 2 + par) * 4;
}
constexpr size_t kP2PBoardBytes = kP2PRedBytes + (size_t)kP2PWMax * 2 * kMailSlot + 512;
// flag value published for a reduction epoch (0 means "not published")
inline unsigned p2p_tag(int64_t epoch) { return (unsigned)(epoch & 0x7fffffff) + 1u; }

State& st();
void require_init();
// store lifecycle and host-synchronising calls cannot be recorded into a graph
// (a relaunch would replay freed memory or stale host buffers): they fail
// while a capture is open
void require_not_capturing(const char* what);
Store& store_of(int64_t sid);
void store_ensure_bytes(Store& s, size_t lo, size_t hi);

// kernels shared across units (dk_kernels.cu)
void launch_accum(const dk_view& target, const double* vals, int64_t stride, int nvals, cudaStream_t s);
void launch_builtin(const std::string& kind, const dk_view* v, int n, const int32_t* writes, cudaStream_t s);
int launch_spmv_csr_dot(const dk_view* v, double* parts, int64_t x_row0, cudaStream_t s);
void launch_fill(double* p, int64_t n, double value, cudaStream_t s);
void launch_timestamp(uint64_t buf, int64_t idx, cudaStream_t s);
void launch_pack(const dk_view& src, double* dst, cudaStream_t s, bool unpack);

inline int64_t view_volume(const dk_view& v) {
  int64_t n = 1;
  for (int d = 0; d < v.rank; ++d) n *= v.ext[d];
  return n;
}

}  // namespace dk
