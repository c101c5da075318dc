/*
 * dk_b200.h -- C ABI of the B200 execution backend for Diffuse fused tasks.
 *
 * The reference has no FFI: its execution path is Python
 * (diffusekit pipeline.py:312-345 Session._execute -> executor.py:163-195
 * execute_task -> kernels.py:717-784 interpret, over the Heap of
 * executor.py:40-79).  This library replaces the *body* of that path; the
 * Python side (paper_2406_18109_b200/runtime.py, ctypes) keeps the
 * reference's call signature and exception types.  Every entry point returns
 * DK_OK (0) or an error code; dk_last_error() describes the last failure of
 * the calling thread.  One process drives one GPU (dk_init); the caller is a
 * single Python thread.
 *
 * Mapping to the reference (file:line of what each group replaces):
 *   dk_store_*      Heap.get / free / digest           executor.py:54-71
 *   dk_kernel_*     interpret (vectorised + per-point)  kernels.py:717-784
 *   dk_launch       execute_task point loop body        executor.py:192-195
 *   dk_builtin      default_builtins MATVEC/SPMV/NORM/OPAQUE  executor.py:93-113
 *                   + SPMV_CSR (new opaque kind)
 *   dk_accum        Rd combine in point order            executor.py:193-195, 287-293
 *   dk_comm_*       (new) halo / replicated-read transfers and partial-sum
 *                   allgather between GPUs (SURVEY §5, §8 e)
 */
#ifndef DK_B200_H
#define DK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DK_OK = 0,
  DK_ERR_CUDA = 1,        /* CUDA runtime / driver failure                      */
  DK_ERR_NVRTC = 2,       /* JIT compilation failed                             */
  DK_ERR_ARG = 3,         /* malformed argument / program                       */
  DK_ERR_OOM = 4,         /* device memory exhausted                            */
  DK_ERR_STATE = 5,       /* not initialised / unknown store or handle          */
  DK_ERR_NCCL = 6,        /* collective failure                                 */
  DK_ERR_PRIVILEGE = 7,   /* store/reduce into a read-only parameter            */
  DK_ERR_BOUNDS = 8,      /* offset access outside a bound sub-store            */
  DK_ERR_UNSUPPORTED = 9  /* shape/broadcast pattern the backend rejects        */
};

enum { DK_F64 = 0, DK_I32 = 1 };

/* A bound sub-store view: element pointer of the view origin plus per-dim
 * extents and element strides (row-major store, innermost stride 1). */
typedef struct {
  uint64_t ptr;
  int32_t rank;
  int32_t dtype;
  int64_t ext[4];
  int64_t stride[4];
} dk_view;

const char* dk_last_error(void);
int dk_version(void);

/* process <-> GPU binding, stream, sync */
int dk_init(int device);
int dk_shutdown(void);
int dk_set_stream(uint64_t stream);        /* 0 = library-owned stream */
int dk_get_stream(uint64_t* stream);
int dk_sync(void);
int dk_device_info(int* sm_count, int64_t* free_bytes, int64_t* total_bytes);
int dk_launch_count(int64_t* count);       /* kernels this library has launched */

/* stores: row-major, VA reserved for the whole store, HBM backed on demand */
int dk_store_create(int64_t sid, int rank, const int64_t* extents, int dtype);
int dk_store_ensure(int64_t sid, int64_t elem_lo, int64_t elem_hi);
int dk_store_free(int64_t sid);
int dk_store_ptr(int64_t sid, uint64_t* dptr);
int dk_store_bytes_mapped(int64_t sid, int64_t* bytes);
/* copy the rect [lo, hi) between a full-store-shaped host array and the store */
int dk_store_upload_rect(int64_t sid, const int64_t* lo, const int64_t* hi, const void* host);
int dk_store_download_rect(int64_t sid, const int64_t* lo, const int64_t* hi, void* host);
int dk_store_fill(int64_t sid, int64_t elem_lo, int64_t elem_hi, double value);

/* Initial contents on the device, bit-identical to numpy's PCG64 streams
 * (Heap.get, executor.py:57-60).  state/inc = {hi, lo} of
 * default_rng(...).bit_generator.state.  dk_pcg64_rejects lists (sorted) the
 * draw indices < draw_end that integers(1, 10) rejects; dk_pcg64_fill writes
 * the rect [lo, hi) of a rank-1/2 f64 store: kind 0 = integers(1, 10) with
 * rejection breakpoints `breaks` (element index after which the draw index
 * shifts by one more), kind 1 = random() * scale. */
int dk_pcg64_rejects(const uint64_t* state, const uint64_t* inc, int64_t draw_end, int64_t* out, int64_t cap,
                     int64_t* count);
int dk_pcg64_fill(int64_t sid, const int64_t* lo, const int64_t* hi, const uint64_t* state, const uint64_t* inc,
                  int kind, double scale, const int64_t* breaks, int64_t nbreaks);

/* scratch (task-local buffers, staging): stream-ordered */
int dk_scratch_alloc(int64_t bytes, uint64_t* dptr);
int dk_scratch_free(uint64_t dptr);
int dk_memset_zero(uint64_t dptr, int64_t bytes);
int dk_memcpy_d2h(void* host, uint64_t dptr, int64_t bytes);   /* synchronising */
int dk_memcpy_h2d(uint64_t dptr, const void* host, int64_t bytes);
int dk_host_alloc(int64_t bytes, void** host);                  /* pinned */
int dk_host_free(void* host);
int dk_memcpy_d2h_async(void* host, uint64_t dptr, int64_t bytes);

/* extra streams / events for host-streamed execution (copy-compute overlap);
 * every enqueueing call uses the current stream (dk_set_stream) */
int dk_stream_new(uint64_t* stream);
int dk_event_new(uint64_t* event);
int dk_event_record(uint64_t event);       /* on the current stream */
int dk_stream_wait_event(uint64_t event);  /* current stream waits */
int dk_event_sync(uint64_t event);
int dk_event_elapsed_ms(uint64_t start, uint64_t stop, float* ms);

/* CUDA graphs (no reference counterpart — the reference re-runs
 * Session._replay, pipeline.py:278-286, per memo hit): capture the library
 * stream's work between begin/end (e.g. one memo-replayed iteration whose
 * launches are prepared) and relaunch it as one graph on the current stream. */
int dk_graph_begin(void);
int dk_graph_end(uint64_t* graph);
int dk_graph_launch(uint64_t graph);
int dk_graph_destroy(uint64_t graph);

/* JIT: program text (paper_2406_18109_b200.ir.KProg.wire) -> handle.
 * Compilation to sm_100a happens at first launch per binding class. */
int dk_kernel_compile(const char* program, int64_t len, int64_t* handle);
int dk_kernel_source(int64_t handle, char* buf, int64_t cap, int64_t* len);
int dk_kernel_num_reductions(int64_t handle, int* n);
/* JIT totals: modules built (one per kernel x binding class), NVRTC compiles,
 * on-disk cubin cache hits (DK_JIT_CACHE), seconds spent in NVRTC */
int dk_jit_stats(int64_t* modules, int64_t* compiles, int64_t* disk_hits, double* seconds);
/* Device-free code generation (and optional NVRTC compile) for a binding:
 * returns the generated CUDA source.  Used by the CPU test-suite. */
int dk_kernel_codegen(const char* program, int64_t len, const dk_view* views, int nviews,
                      const double* scalars, int compile, char* buf, int64_t cap, int64_t* out_len);

/* Run one launch point.  views[i] binds slot i.  totals == 0: every reduce
 * statement accumulates into its target view in statement order; otherwise
 * the per-statement totals are written to totals[k] (multi-GPU fold). */
int dk_launch(int64_t handle, const dk_view* views, int nviews,
              const double* scalars, int nscalars, uint64_t totals);

/* for i in 0..nvals-1: target[...] += vals[first + i*stride]  (device values, in order) */
int dk_accum(const dk_view* target, uint64_t vals, int64_t first, int64_t stride, int nvals);

/* opaque kinds: kind = "MATVEC" | "SPMV" | "NORM" | "OPAQUE" | "SPMV_CSR" */
int dk_builtin(const char* kind, const dk_view* views, int nviews, const int32_t* writes);

/* SPMV_CSR with the opt-in partial-dot epilogue (DK_FUSE_SPMV_DOT=1; backend-only, it
 * changes which launch computes the following window's p.q, never the fusion plan):
 * views as dk_builtin("SPMV_CSR"); also writes per-CTA partials of sum_i x[x_row0+i]*y[i]
 * (i over this tile's rows, each partial a fixed in-order sum) to parts[0 .. *nparts) and,
 * from the last CTA, their fixed-order fold to parts[DK_SPMV_DOT_TOTAL].  `parts`: device,
 * DK_SPMV_DOT_DOUBLES doubles; the 32-bit ticket at parts[DK_SPMV_DOT_PARTS] must be zero on
 * entry (the kernel leaves it zero).  Replaces, for that window, the DOT(p, q -> pq)
 * reduction of the cg_like stream (trace.py:384-386). */
#define DK_SPMV_DOT_PARTS 4096
#define DK_SPMV_DOT_TOTAL (DK_SPMV_DOT_PARTS + 1)
#define DK_SPMV_DOT_DOUBLES (DK_SPMV_DOT_PARTS + 2)
int dk_spmv_csr_dot(const dk_view* views, uint64_t parts, int64_t x_row0, int* nparts);

/* multi-GPU (NCCL over NVLink/NVSwitch); one rank per process */
int dk_comm_unique_id(uint8_t* out128);
int dk_comm_init(int rank, int world, const uint8_t* id128);
int dk_comm_destroy(void);
/* grouped point-to-point moves of store rects; dir: 0 send, 1 recv */
int dk_comm_exchange(int n, const int64_t* sids, const int32_t* peers, const int32_t* dirs,
                     const int64_t* los, const int64_t* his);
/* allgather `count` doubles per rank from device ptr src into dst (world*count) */
int dk_comm_allgather_f64(uint64_t src, uint64_t dst, int64_t count);
int dk_comm_barrier(void);

/* Peer-memory reduction exchange (replaces dk_comm_allgather_f64 for fused
 * kernel reductions; no reference counterpart -- the reference combines
 * per-point arenas in one host heap, executor.py:193-195).  Every rank owns a
 * small "board" (DK_P2P_SLOTS ring slots of [world][DK_P2P_POINTS][DK_P2P_RED]
 * doubles plus one flag per (rank, point)); the boards are IPC-mapped on every
 * rank, so a reducing kernel's last CTA writes its point's per-statement
 * totals straight into every rank's board over NVLink and raises the matching
 * flag there -- the compute step and the all-gather are one kernel. */
#define DK_P2P_SLOTS 4
#define DK_P2P_POINTS 16
#define DK_P2P_RED 32
/* diagnostics: a one-thread kernel writes %globaltimer (ns) to ((uint64_t*)buf)[idx] when the
 * stream reaches it -- per-rank device timelines of the multi-GPU step (bench DK_TRACE_TS) */
int dk_timestamp(uint64_t buf, int64_t idx);
/* collective (after dk_comm_init): *enabled = 1 iff every rank mapped every peer's board */
int dk_p2p_init(int* enabled);
/* dk_launch with totals published to all ranks' boards for reduction number
 * `epoch` (0, 1, 2, ... in the same order on every rank; ring slot epoch mod
 * DK_P2P_SLOTS), `point` = ordinal of this launch point among the calling
 * rank's points.  The flag raised in each board holds the epoch's tag
 * (epoch mod 2^31, + 1), so a consumer can tell this epoch's totals from an
 * older or newer use of the slot. */
int dk_launch_pub(int64_t handle, const dk_view* views, int nviews, const double* scalars, int nscalars,
                  int64_t epoch, int point);
/* dk_launch_pub whose point block holds nred_total totals of which the kernel writes
 * its own at [red_offset, red_offset + its reductions): the rest of the block was filled
 * earlier on the stream (dk_p2p_block) -- how the opt-in SpMV + partial-dot epilogue
 * publishes the SpMV's p.q total with the following window's reductions (the
 * DOT(p, q -> pq) of trace.py:384-386, combined in point order as executor.py:193-195). */
int dk_launch_pub_ex(int64_t handle, const dk_view* views, int nviews, const double* scalars, int nscalars,
                     int64_t epoch, int point, int red_offset, int nred_total);
/* device address of this rank's block for `point` in the board slot of `epoch`
 * (nred_total doubles) */
int dk_p2p_block(int64_t epoch, int point, int nred_total, uint64_t* ptr);
/* stream-ordered wait until counts[q] points of every rank q have published
 * epoch `epoch` into this rank's board (flags consumed); a flag holding any
 * other epoch's tag is a protocol violation and traps; *gathered = the slot's
 * totals, layout [world][DK_P2P_POINTS][nred] as dk_accum's `vals` */
int dk_p2p_wait(int64_t epoch, const int32_t* counts, uint64_t* gathered);
/* dk_p2p_wait and the point-order fold in one kernel: after the flags, the
 * kernel applies, in order, target[f] = target[f] + g[first[f] + k*stride[f]]
 * for k < n[f] (g = the slot's gathered totals) to nfold (<= DK_P2P_FOLDS)
 * scalar targets (device pointers to fp64) -- what dk_accum would do per fold,
 * without the extra launches on the reduction's critical path. */
#define DK_P2P_FOLDS 64
int dk_p2p_wait_fold(int64_t epoch, const int32_t* counts, int nfold, const uint64_t* targets,
                     const int64_t* firsts, const int64_t* strides, const int32_t* ns);

/* Halo / replicated-read moves over peer memory instead of NCCL send/recv
 * (same arguments as dk_comm_exchange).  Each rank's board also holds a
 * mailbox per (source rank, parity) of DK_P2P_MAIL_BYTES: one kernel packs
 * this rank's send rects straight into the receivers' mailboxes over NVLink
 * and raises a flag there (tag of the k-th message from this rank to that
 * peer); its receive CTAs wait for the senders' flags, unpack into the store
 * rects and acknowledge, so a sender reuses a mailbox parity only after the
 * receiver consumed the message two before.  The per-direction message
 * counts live in the library (process lifetime), so every pair of ranks
 * agrees on them as long as both call this for the pair's moves.  Fails with
 * DK_ERR_UNSUPPORTED if one pair's bytes exceed a mailbox; the caller then
 * uses dk_comm_exchange (the decision is the same on both ranks). */
#define DK_P2P_MAIL_BYTES (1 << 20)
int dk_p2p_exchange(int n, const int64_t* sids, const int32_t* peers, const int32_t* dirs, const int64_t* los,
                    const int64_t* his);
/* The same mailbox protocol driven by copy engines and stream memory operations
 * (no SMs), so a halo can move while a persistent kernel owns the SMs:
 * dk_dma_send -- on the current stream: per peer, wait (cuStreamWaitValue32)
 * for the receiver's ack of the message two before, copy the (contiguous)
 * rects into its mailbox over NVLink (cudaMemcpyAsync), then write the
 * message tag into its mail flag (cuStreamWriteValue32, fenced);
 * dk_dma_recv -- on the current stream: per peer, wait for the tag, copy the
 * mailbox into the store rects, write the ack into the sender's board.
 * dirs are implied (all sends / all receives); counters shared with
 * dk_p2p_exchange. */
int dk_dma_send(int n, const int64_t* sids, const int32_t* peers, const int64_t* los, const int64_t* his);
int dk_dma_recv(int n, const int64_t* sids, const int32_t* peers, const int64_t* los, const int64_t* his);

#ifdef __cplusplus
}
#endif
#endif
