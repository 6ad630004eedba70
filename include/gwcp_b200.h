/*
 * gwcp_b200.h — C-ABI of the B200-native G-WCP trace-analysis engine.
 *
 * The reference (gpurace 0.1.0, pure Python) has no FFI: its hot path is the
 * duck-typed detector protocol driven by
 *     engine.run(trace, GwcpDetector(cfg))          pkg/src/gpurace/engine.py:98-155
 * and the CLI front end
 *     gpurace check TRACE --detector gwcp           pkg/src/gpurace/cli.py:63-84
 * Every entry point below replaces one piece of that path; the Python shim in
 * paper_2111_12478_b200/ (engine.run / GwcpDetector / cli) binds them with
 * ctypes, and INTEGRATION.md shows the stub a gpurace maintainer would add.
 *
 * Conventions: plain pointers and sizes only; 0 = success, non-zero = error
 * with a message in gw_last_error(); nothing is silently truncated; arrays in
 * a gw_trace / gw_result are owned by the library and released by the
 * matching *_free call.  One analysis per context at a time (not reentrant per
 * context); distinct contexts may be used from distinct host threads.
 */
#ifndef GWCP_B200_H
#define GWCP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GW_OK 0
#define GW_E_PARSE 1        /* text trace rejected (TraceParseError, trace.py:142-145) */
#define GW_E_UNSUPPORTED 2  /* value outside the SoA encoding (e.g. addr >= 2^63, >2^24 threads) */
#define GW_E_CUDA 3         /* CUDA runtime / kernel error */
#define GW_E_NOMEM 4        /* device or host allocation failed */
#define GW_E_ARG 5          /* bad arguments */

/* ---- SoA event encoding (16 B / event) ---------------------------------
 * tidop  : bits 0-23 flat thread index (b*W + w)*L + l      (trace.py:105-106)
 *          bits 24-26 kind, bit 27 atomic, bit 28 device scope,
 *          bit 29 warp barrier, bit 30 continues-record (same group as the
 *          previous event, group >= 0; engine.py:111-118)
 *          barriers carry the flat index of lane 0 of their warp / block.
 * key    : access  -> location key: global addr (< 2^63), or
 *                     1<<63 | block<<40 | addr (addr < 2^40) for shared memory
 *          acq/rel -> lock id (u64)
 * instr  : access  -> instruction id (u32); warp barrier -> lane mask
 */
#define GW_K_READ 0u
#define GW_K_WRITE 1u
#define GW_K_ACQUIRE 2u
#define GW_K_RELEASE 3u
#define GW_K_BARRIER 4u
#define GW_K_FENCE 5u
#define GW_K_END 6u
#define GW_OP_SHIFT 24
#define GW_TID_MASK 0x00FFFFFFu
#define GW_F_ATOMIC (1u << 27)
#define GW_F_DEVICE (1u << 28)
#define GW_F_WARPBAR (1u << 29)
#define GW_F_CONT (1u << 30)
#define GW_SHARED_BIT (1ull << 63)

/* report kinds (report.py:13-15) */
#define GW_WW 0
#define GW_WR 1
#define GW_RW 2

/* diagnostic codes (gwcp.py:178-182, :197-201, :323-330) */
#define GW_D_REENTRANT 1
#define GW_D_UNHELD 2
#define GW_D_EXIT_HOLDING 3

typedef struct gw_config {
  uint32_t blocks, warps, lanes, _pad; /* TraceConfig, trace.py:95-106 */
} gw_config;

typedef struct gw_trace { /* library-owned host SoA (gw_parse_text) */
  gw_config cfg;
  uint64_t n_events;
  uint64_t* key;
  uint32_t* tidop;
  uint32_t* instr;
} gw_trace;

typedef struct gw_trace_view { /* caller-owned SoA; host or device pointers */
  gw_config cfg;
  uint64_t n_events;
  const uint64_t* key;
  const uint32_t* tidop;
  const uint32_t* instr;
} gw_trace_view;

#define GW_OPT_EAGER 1u   /* never capture / replay a CUDA graph for this analysis */
#define GW_OPT_PROFILE 2u /* eager, with CUDA events around every launch (gw_ctx_kernel_times) */
#define GW_OPT_HB 4u      /* scoped happens-before detector (gpurace check --detector hb, hb.py) */

typedef struct gw_opts {
  uint32_t inactive_opt; /* GwcpDetector(inactive_opt=...), gwcp.py:108-127 */
  uint32_t flags;        /* GW_OPT_* */
  void* stream;          /* cudaStream_t to launch on (NULL = legacy default; never graph-replayed) */
  /* Address sharding (multi-GPU): this call reports only the races whose
   * location lies in contiguous location-key range shard_index of
   * shard_count (0 or 1 = unsharded).  Every shard holds the whole trace and
   * runs the sync pass; dedup is shard-local because the dedup key contains
   * the location (report.py:93), so concatenating the shards' reports and
   * ordering them by order_key gives the unsharded result (report 0 is the
   * global "first"). */
  uint32_t shard_index;
  uint32_t shard_count;
} gw_opts;

typedef struct gw_result { /* library-owned; reports in final order */
  uint64_t n_reports;      /* report 0 is "first", the rest "post-race" (report.py:97) */
  uint8_t* kind;           /* GW_WW / GW_WR / GW_RW */
  uint32_t* prior_event;   /* event indices; tid/instr/loc are read from the trace */
  uint32_t* current_event;
  uint64_t n_diags;        /* in event order */
  uint32_t* diag_event;
  uint32_t* diag_code;     /* GW_D_* */
  uint64_t* diag_lock;     /* lock id (EXIT_HOLDING: one entry per held frame, bottom->top) */
  uint64_t* order_key;     /* per report: (record-head or current event) << 32 | sub-order; increasing */
} gw_result;

typedef struct gw_stats { /* per-phase device times of the last analysis (ms) */
  float ms_total, ms_prep, ms_walker, ms_sort, ms_check, ms_final;
  uint64_t n_accesses, n_candidates, n_sync, arena_words;
  uint32_t walker_ctas, sort_bits;
  uint64_t n_sorted;       /* positions the access pass sorted (all events, or this shard's accesses) */
} gw_stats;

typedef struct gw_ctx gw_ctx;

/* ---- host-side trace ingest (replaces parse_trace, trace.py:226-398) ---- */
int gw_parse_text(const char* text, uint64_t len, gw_trace* out, int64_t* err_line);
void gw_trace_free(gw_trace* t);

/* Binary SoA trace file (the on-disk form of the
 * columnar trace, 16 B/event, loaded without parsing).  Little-endian layout:
 *   magic "GWSOA\0\1\0" (8 B) | blocks, warps, lanes, reserved (4 x u32) |
 *   n_events (u64) | key[n] (u64) | tidop[n] (u32) | instr[n] (u32)
 * gw_load_soa checks the header, the file size and that every event's
 * thread index and kind are inside the configured hierarchy / encoding
 * (GW_E_PARSE otherwise); it does not run validate_trace. */
int gw_save_soa(const char* path, const gw_trace_view* t);
int gw_load_soa(const char* path, gw_trace* out);

/* validate_trace (trace.py:522-601): diagnostics as (event, code, a, b); see cli shim */
int gw_validate(const gw_trace_view* t, uint64_t* n_out, uint32_t** ev, uint32_t** code,
                uint64_t** a, uint64_t** b);
void gw_free(void* p);

/* validate_trace on the GPU: same diagnostics, codes
 * and order as gw_validate, computed with per-thread segmented passes
 * (first END per thread, per-event / per-barrier checks, lock stacks walked
 * per thread over the tid-sorted lock events).  host_trace: host SoA. */
int gw_ctx_validate(gw_ctx* c, const gw_trace_view* host_trace, uint64_t* n_out, uint32_t** ev, uint32_t** code,
                    uint64_t** a, uint64_t** b);
/* infer_locks (trace.py:609-680) on the GPU: the rewritten trace (out, free
 * with gw_trace_free) and one diagnostic per release left uninferred
 * (event index in the INPUT trace, lock, thread), in the reference's order:
 * thread by thread (threads by first event), then by event. */
int gw_ctx_infer_locks(gw_ctx* c, const gw_trace_view* host_trace, gw_trace* out, uint64_t* n_diag,
                       uint32_t** diag_event, uint64_t** diag_lock, uint32_t** diag_tid);

/* ---- analysis (replaces engine.run + GwcpDetector, engine.py:98-155, gwcp.py:103-356) */
/* host SoA in, host results out: H2D, all kernels, D2H inside */
int gw_analyze(const gw_trace_view* host_trace, const gw_opts* opts, gw_result* out);
void gw_result_free(gw_result* r);
const char* gw_last_error(void);

/* device-resident context API: buffers persist across calls.  Lock-free
 * traces analysed repeatedly with the same shape, input buffers and
 * (non-default) stream are replayed from a captured CUDA graph; the plan is
 * re-verified on the device and a mismatch falls back to an eager run inside
 * gw_ctx_fetch, so results never depend on the cache. */
gw_ctx* gw_ctx_create(int device);
void gw_ctx_destroy(gw_ctx* c);
/* dev_trace points at device memory; enqueues on opts->stream; results stay on device.
 * The dev_trace buffers must stay valid and unmodified until the matching
 * gw_ctx_fetch returns: a graph replay whose plan check fails is re-run
 * eagerly inside gw_ctx_fetch, reading them again. */
int gw_ctx_analyze_device(gw_ctx* c, const gw_trace_view* dev_trace, const gw_opts* opts);
/* host_trace in (pageable or pinned) -> H2D on opts->stream -> analyze (results on device) */
int gw_ctx_analyze_host(gw_ctx* c, const gw_trace_view* host_trace, const gw_opts* opts);
/* ---- exchange mode: the multi-GPU data plane (paper_2111_12478_b200/shard.py)
 * Every rank holds ONE record-aligned slice of the trace (1/G of the SoA,
 * device pointers) at global event offset event_base; the host moves the
 * data between ranks with NCCL collectives:
 *   gw_xs_prep       slice statistics -> the host sums / ORs / ANDs them
 *   gw_xs_hard       the slice's barriers and ENDs (global event, tidop,
 *                    instr, key) -> all-gathered: every rank runs the small
 *                    sync pass (snapshot walker) over the whole trace's
 *   gw_xs_partition  the slice's accesses as 12-byte records (h, global
 *                    event | W, tidop) grouped by destination shard = the
 *                    top log2(G) bits of h = fmix32(compacted location) ->
 *                    all-to-all
 *   gw_xs_check      the bucketed check of this shard's received records,
 *                    plus the record (same-instruction) check of the slice;
 *                    gw_xs_fetch the candidates (global event indices)
 *   gw_xs_lookup     (tidop, instr) of global events in the slice, for the
 *                    report merge on rank 0 (dedup report.py:92-100 is per
 *                    location, so any partition of the locations is exact).
 * Lock-free traces with records of <= 32 events; a shard meeting hot
 * locations or > 32-read windows returns GW_E_UNSUPPORTED (the host then
 * uses the replicated address-sharded mode of gw_opts). */
typedef struct gw_xs_stats {
  uint64_t n_acc, n_write, n_acq, n_rel, n_end, n_bar, key_or, key_and, n_long, n_wbar;
} gw_xs_stats;
int gw_xs_prep(gw_ctx* c, const gw_trace_view* dev_slice, uint32_t event_base, void* stream, gw_xs_stats* out);
int gw_xs_hard(gw_ctx* c, void* stream, uint32_t* ev, uint32_t* tidop, uint32_t* instr, uint64_t* key,
               uint64_t* n_out);
int gw_xs_partition(gw_ctx* c, const gw_xs_stats* global, uint32_t shard_count, void* stream, uint32_t* h,
                    uint32_t* v, uint32_t* t, uint64_t* counts);
int gw_xs_check(gw_ctx* c, const gw_xs_stats* global, uint32_t shard_count, uint64_t n_total, void* stream,
                const uint32_t* h, const uint32_t* v, const uint32_t* t, uint64_t n_recv, const uint32_t* hev,
                const uint32_t* htidop, const uint32_t* hinstr, const uint64_t* hkey, uint64_t n_hard,
                uint64_t* n_cand);
int gw_xs_fetch(gw_ctx* c, uint64_t* okey, uint64_t* loc, uint32_t* prior, uint32_t* cur, uint32_t* kind);
int gw_xs_lookup(gw_ctx* c, const uint32_t* ev, uint64_t n, uint32_t* tidop, uint32_t* instr);

/* Packed (narrow-column) trace: the SoA above with the key column stored in
 * key_bytes = 4 or 8 and the instr column in instr_bytes = 2 or 4 bytes per
 * event -- the narrowest widths holding every value of the trace (C5:
 * 10 B/event instead of 16).  Barrier keys are implied by their tidop
 * (warp barrier: block << 32 | warp; block barrier: 0): with 4-byte keys
 * they are not stored (any value) and are restored on the device.  It is the layout of GWSOA v2 files (cli
 * convert --packed) and the host input of gw_ctx_analyze_host_packed, which
 * uploads it in chunks on a copy stream and widens each chunk on the device
 * while the next one is in flight, then analyses as gw_ctx_analyze_host. */
typedef struct gw_trace_packed {
  gw_config cfg;
  uint64_t n_events;
  uint32_t key_bytes, instr_bytes;
  const void* key;        /* uint32_t[n] (key_bytes 4) or uint64_t[n] */
  const uint32_t* tidop;
  const void* instr;      /* uint16_t[n] (instr_bytes 2) or uint32_t[n] */
} gw_trace_packed;
int gw_ctx_analyze_host_packed(gw_ctx* c, const gw_trace_packed* host_trace, const gw_opts* opts);
/* Delta-varint trace (GWSOA v3): per column (0 key u64, 1 tidop u32,
 * 2 instr u32) the differences of consecutive events, zigzag-coded LEB128
 * varints; chunks of GW_DELTA_CHUNK events start at offs[c][k] and decode
 * on their own from base[c][k] = the column's value before the chunk.
 * Consecutive lanes of a record differ by small constants, so the C2 / C5
 * traces take ~3.3 B/event.  gw_encode_delta builds it on the host (chunk-
 * parallel; library-owned arrays, gw_delta_free); gw_ctx_analyze_host_delta
 * uploads the three byte streams in slices on a copy stream while the
 * device decodes the slices already landed (k_delta_decode), then analyses
 * as gw_ctx_analyze_host. */
#define GW_DELTA_CHUNK 4096u
typedef struct gw_trace_delta {
  gw_config cfg;
  uint64_t n_events;
  uint32_t chunk, _pad;
  uint64_t n_chunks;
  const uint8_t* bytes[3];
  uint64_t nbytes[3];
  const uint64_t* offs[3]; /* n_chunks + 1 */
  const uint64_t* base[3]; /* n_chunks */
} gw_trace_delta;
int gw_encode_delta(const gw_trace_view* host_trace, gw_trace_delta* out);
void gw_delta_free(gw_trace_delta* d);
int gw_ctx_analyze_host_delta(gw_ctx* c, const gw_trace_delta* host_trace, const gw_opts* opts);
/* Bit-packed trace (GWSOA v4): per column (0 key u64, 1 tidop u32, 2 instr
 * u32) and chunk of GW_DELTA_CHUNK events, blocks of 32 values.  A block
 * stores the residuals of the column's first differences d_i = x_i - x_{i-1}
 * (mod 2^w) against a prediction -- d_{i-1} (mode 0), d_{i-32} (mode 1),
 * d_{i-64} (mode 2; warp-structured traces repeat every 32-lane record, or
 * every other one) or 0 (mode 3); modes 1 / 2 need 1 / 2 earlier blocks of
 * the chunk -- zigzag-coded and packed at the block's width b bits (0..31),
 * the residuals wider than b as exceptions.  Chunk k's bytes (from
 * offs[c][k], 4-byte aligned): hdr[nb] (bits 7-6 mode, bit 5 has exceptions,
 * bits 0-4 b; nb = ceil(events / 32)), per block with exceptions a count
 * byte and a value-width byte xw, zero pad to 4, b little-endian 32-bit words
 * per block (lane l's bits at l * b), the exceptions' lane bytes, their
 * zigzag values (xw bytes each, little endian), zero pad to 4.  base[c][k] /
 * dbase[c][k]: the column's value and first difference before chunk k.
 * C5: ~0.3 B/event instead of 3.3.  gw_encode_bp builds it on the host
 * (chunk-parallel, gw_bp_free); gw_ctx_analyze_host_bp uploads it in slices
 * and decodes each slice on the device (one warp per chunk and column)
 * while the next is in flight. */
typedef struct gw_trace_bp {
  gw_config cfg;
  uint64_t n_events;
  uint32_t chunk;
  uint32_t key_bits;        /* 32: every key < 2^32, column 0 coded as a 32-bit column; else 64 */
  uint64_t n_chunks;
  const uint8_t* bytes[3];
  uint64_t nbytes[3];
  const uint64_t* offs[3];  /* n_chunks + 1 */
  const uint64_t* base[3];  /* n_chunks */
  const uint64_t* dbase[3]; /* n_chunks */
} gw_trace_bp;
int gw_encode_bp(const gw_trace_view* host_trace, gw_trace_bp* out);
void gw_bp_free(gw_trace_bp* t);
int gw_ctx_analyze_host_bp(gw_ctx* c, const gw_trace_bp* host_trace, const gw_opts* opts);
/* D2H of the last analysis' results (synchronises the stream) */
int gw_ctx_fetch(gw_ctx* c, gw_result* out);
int gw_ctx_stats(gw_ctx* c, gw_stats* out);
/* number of kernels the last analysis launched */
uint32_t gw_ctx_launches(gw_ctx* c);
/* per-kernel device times of the last GW_OPT_PROFILE analysis (aggregated by kernel) */
int gw_ctx_kernel_times(gw_ctx* c, uint32_t cap, char (*names)[64], float* ms, uint32_t* launches, uint32_t* n_out);

/* bench / test infrastructure: generate the C2 / C5 synthetic trace (SURVEY
 * §8(d)) directly into device buffers of phases*(records*B*W*L + B) events */
int gw_gen_c2_device(uint32_t blocks, uint32_t warps, uint32_t lanes, uint32_t phases, uint32_t records,
                     uint64_t words_per_block, uint64_t seed, uint64_t* key, uint32_t* tidop, uint32_t* instr,
                     void* stream);
/* C4 (ITS divergence, lanes = 32): iters*(B*W*32) accesses + B*W*(iters/4) warp
 * barriers + B*(iters/64) block barriers */
int gw_gen_c4_device(uint32_t blocks, uint32_t warps, uint32_t iters, uint64_t words_per_block, uint64_t seed,
                     uint64_t* key, uint32_t* tidop, uint32_t* instr, void* stream);

/* C3 (spin locks, lanes <= 32): group_offsets[g] (device, u64) = first event of
 * group g = (it*B + b)*W + w, from workloads.c3_group_offsets */
int gw_gen_c3_device(uint32_t blocks, uint32_t warps, uint32_t lanes, uint32_t iters, uint32_t locks,
                     uint32_t region, uint32_t priv, uint64_t seed, const uint64_t* group_offsets, uint64_t* key,
                     uint32_t* tidop, uint32_t* instr, void* stream);

#ifdef __cplusplus
}
#endif
#endif
