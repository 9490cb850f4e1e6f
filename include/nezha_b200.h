/*
 * nezha_b200.h — C ABI of the B200-native multi-rail allreduce.
 *
 * Plain C: opaque handles, plain pointers and sizes, int return codes
 * (0 = ok, < 0 = error, message in nz_last_error()). Nothing throws across
 * this boundary and no torch type appears in it. One process drives one GPU,
 * or (nz_comm_init_loopback) one host thread drives one virtual rank of a job
 * whose ranks all live on one GPU.
 *
 * Which reference interface each group replaces (file:line under
 * /root/reference):
 *   nz_comm_*      rendezvous(TransportOptions) -> ConnectionSet
 *                  (proj/include/nezha/transport/transport.hpp:219-238) and
 *                  FileStore (proj/include/nezha/transport/rendezvous.hpp:19-37):
 *                  the per-rank bootstrap that builds the full rail mesh.
 *   nz_buffer_*    UnboundBuffer: the shared
 *                  reduction buffer every rail reads its segment from.
 *   nz_rail_*      one rail's ring_allreduce / ring_chunked_allreduce over its
 *                  segment on top of Channel::send/recv
 *                  (transport.hpp:89-123); failure injection replaces
 *                  InMemoryFabric::failRailAtFrame (inmem.hpp:22-24).
 *   nz_engine_*    the engine-level multi-rail allreduce (SPEC.md:226, :353,
 *                  :416; named by proj/tests/CMakeLists.txt:17): allocate ->
 *                  per-rail executors -> join -> Timer -> balancer -> handoff.
 *   nz_planner_*   the balancer + faults decisions alone,
 *                  trace driven, CPU only; what the parity tests diff.
 *   nz_pool_*      ComputePool: per-phase
 *                  compute tokens; on B200 the tokens are SMs (P14).
 *   nz_core_*      core cost model (proj/include/nezha/core/math.hpp:9-17,
 *                  types.hpp:26-44) for FFI callers without C++.
 */
#ifndef NEZHA_B200_H
#define NEZHA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NZ_ABI_VERSION 3

enum {
  NZ_OK = 0,
  NZ_ERR_INVALID = -1,      /* std::invalid_argument in the C++ API */
  NZ_ERR_CUDA = -2,         /* a CUDA runtime / driver call failed */
  NZ_ERR_SYSTEM = -3,       /* socket / fd / OS failure during bootstrap */
  NZ_ERR_UNSUPPORTED = -4,  /* e.g. NVLS rail without multicast support */
  NZ_ERR_RAIL_DOWN = -5,    /* ChannelDownError */
  NZ_ERR_UNRECOVERABLE = -6,/* UnrecoverableError: no surviving rail */
  NZ_ERR_TIMEOUT = -7,      /* RendezvousTimeoutError / device watchdog */
  NZ_ERR_BUFFER = -8        /* output buffer too small */
};

typedef enum { NZ_F32 = 0, NZ_BF16 = 1, NZ_I32 = 2 } nz_dtype_t;

/* B200 rails. Protocol names in rails TOML: sharp|nvls, glex|ce, tcp|sm. */
typedef enum { NZ_RAIL_NVLS = 0, NZ_RAIL_CE = 1, NZ_RAIL_SM = 2 } nz_rail_kind_t;

typedef enum { NZ_ALGO_RING = 0, NZ_ALGO_RING_CHUNKED = 1 } nz_algorithm_t;

typedef struct nz_comm nz_comm_t;
typedef struct nz_buf nz_buf_t;
typedef struct nz_rail nz_rail_t;
typedef struct nz_engine nz_engine_t;

const char* nz_last_error(void);
int nz_abi_version(void);
/* sizeof of the ABI's structs for FFI bindings that lay them out themselves:
 * "engine_config", "failover_report", "rail_status", "fault_record";
 * NZ_ERR_INVALID for another name. */
int nz_abi_sizeof(const char* type_name);
/* 1 when this build contains the sm_100a kernels (always, for the product). */
int nz_has_cuda_kernels(void);

/* ---------------------------------------------------------------- comm --- */
/* Bootstrap of one rank (one GPU). `session` names the rendezvous: every rank
 * of one job passes the same string (e.g. "<MASTER_PORT>-<job>"). File
 * descriptors for peer memory and the multicast object travel over abstract
 * unix sockets, the FileStore analogue. Blocks until all ranks arrive or
 * `timeout_ms` passes (NZ_ERR_TIMEOUT). */
int nz_comm_init(int rank, int world, int device, const char* session, int timeout_ms, nz_comm_t** out);
/* Loopback bootstrap of one VIRTUAL rank: `world` ranks of one job live in
 * this process on the same `device`, one host thread per rank, each calling
 * this with the same `session`. Buffers are per-rank allocations on that GPU
 * whose pointers are exchanged in process; every cross-rank kernel runs all
 * virtual ranks in one grid (blockIdx.y = rank) sized to be co-resident, so
 * the rails' exact protocols (barriers, LL flags, copy-engine DMA between
 * ranks' memory, failure detection) run on a single B200. No multicast, so
 * no NVLS rail. Every other entry point is used exactly as with nz_comm_init. */
int nz_comm_init_loopback(int rank, int world, int device, const char* session, int timeout_ms, nz_comm_t** out);
int nz_comm_is_loopback(const nz_comm_t* comm);
/* Loopback only: marks the job's virtual-rank group failed (a rank's host
 * code raised), so every peer waiting in an exchange or a combined launch
 * fails at once (NZ_ERR_TIMEOUT) instead of after `timeout_ms`. NZ_OK and no
 * effect on a multi-process comm. */
int nz_comm_abort(nz_comm_t* comm);
int nz_comm_destroy(nz_comm_t* comm);
int nz_comm_rank(const nz_comm_t* comm);
int nz_comm_world(const nz_comm_t* comm);
int nz_comm_device(const nz_comm_t* comm);
int nz_comm_sm_count(const nz_comm_t* comm);
int nz_comm_multicast_supported(const nz_comm_t* comm);
/* Host-side barrier and allgather of small host blobs (`all` holds world*bytes). */
int nz_comm_barrier(nz_comm_t* comm);
int nz_comm_allgather(nz_comm_t* comm, const void* mine, size_t bytes, void* all);

/* -------------------------------------------------------------- buffers --- */
/* Symmetric device buffer: the same size on every rank, mapped into every
 * rank's address space (peer pointers) and bound to a multicast object when
 * the fabric supports it. Collective: all ranks call with the same size. */
int nz_buffer_alloc(nz_comm_t* comm, size_t bytes, nz_buf_t** out);
int nz_buffer_free(nz_buf_t* buf);
void* nz_buffer_ptr(const nz_buf_t* buf);
void* nz_buffer_peer_ptr(const nz_buf_t* buf, int rank);
void* nz_buffer_mc_ptr(const nz_buf_t* buf); /* NULL without multicast */
size_t nz_buffer_size(const nz_buf_t* buf);
/* Copy into / out of this rank's part of the buffer. `src` / `dst` may be
 * host (pinned or pageable) or device memory. With stream == NULL the copy is
 * synchronous; otherwise it is enqueued on `stream`. */
int nz_buffer_write(nz_buf_t* buf, uint64_t offset, const void* src, uint64_t bytes, void* stream);
int nz_buffer_read(const nz_buf_t* buf, uint64_t offset, void* dst, uint64_t bytes, void* stream);
int nz_buffer_fill_zero(nz_buf_t* buf, void* stream);

/* ---------------------------------------------------------------- rails --- */
/* A rail owns a CUDA stream on this rank, its barrier pads and (CE) staging.
 * `sm_budget` caps the CTAs its kernels use (0 = all SMs). */
int nz_rail_create(nz_comm_t* comm, int kind, int rail_id, int sm_budget, nz_rail_t** out);
/* NZ_RAIL_FLAG_GRAPH_SAFE: the rail's kernels take their barrier epochs and
 * LL flags from a device counter (advanced by the last CTA of each launch)
 * instead of launch arguments, so its launches can be captured in a CUDA
 * graph and replayed any number of times, mixed with eager calls. Collective
 * (all ranks pass the same flags). Warm up once before capturing (the CE rail
 * sizes its staging buffer on first use). */
#define NZ_RAIL_FLAG_GRAPH_SAFE 1
int nz_rail_create_ex(nz_comm_t* comm, int kind, int rail_id, int sm_budget, int flags, nz_rail_t** out);
int nz_rail_destroy(nz_rail_t* rail);
int nz_rail_kind(const nz_rail_t* rail);
/* Blocks the host until all work enqueued on the rail's own streams is done. */
int nz_rail_synchronize(nz_rail_t* rail);
void* nz_rail_stream(const nz_rail_t* rail);

/* Allreduce chunks [chunk_begin, chunk_end) of the segment geometry
 * (seg_off, seg_len, chunk_bytes) from `in` into `out` (out-of-place; in ==
 * out is allowed when no failure injection is armed). Enqueued on `stream`
 * (NULL = the rail's own stream); returns without waiting. Summation order:
 * DESIGN.md P1 (CE, SM: exact; NVLS: switch order). If `fail_chunk` lies in
 * [chunk_begin, chunk_end) the rail stops before that chunk on every rank and
 * posts a fault record (nz_rail_poll_fault): deterministic injection of the
 * trace form (op_seq, rail, chunk k), P10. -1 disables it. */
int nz_rail_allreduce(nz_rail_t* rail, nz_buf_t* in, nz_buf_t* out, uint64_t seg_off, uint64_t seg_len,
                      uint64_t chunk_bytes, uint64_t chunk_begin, uint64_t chunk_end, int dtype,
                      uint32_t op_seq, int64_t fail_chunk, void* stream);

/* Trace-form failure for the rail's next nz_rail_allreduce on this rank: the
 * same as passing fail_chunk = chunk to it (InMemoryFabric::failRailAtFrame,
 * inmem.hpp:22-24). Every rank arms the same chunk. */
int nz_rail_inject_failure(nz_rail_t* rail, uint64_t chunk);
/* Chunks of the last nz_rail_allreduce that are complete on this rank, from
 * the device progress record: a call runs as waves of consecutive chunks
 * (one launch each, >= 32 MiB apiece) and each wave that succeeds publishes
 * its end chunk, so the count moves from chunk_begin through the wave ends to
 * the stop chunk (chunk_end, or the injected trace-form failure chunk).
 * Non-blocking. */
int nz_rail_progress(nz_rail_t* rail, uint64_t* chunks_done);
/* Kills the rail on this rank (InMemoryFabric::killRail, inmem.cpp:214-233):
 * later nz_rail_allreduce calls fail with NZ_ERR_RAIL_DOWN. Work already on
 * the device cannot be preempted: it completes, or its cross-rank waits are
 * bounded by the watchdog when a peer never arrives. */
int nz_rail_abort(nz_rail_t* rail);
/* Elapsed microseconds between two recorded cudaEvent_t (e.g. around a rail
 * call on its stream), for FFI callers without the CUDA runtime. */
int nz_event_elapsed_us(void* start_event, void* end_event, double* us);

typedef struct {
  uint32_t valid;      /* 1 once the device posted a fault */
  uint32_t op_seq;
  uint64_t chunk;      /* first chunk NOT completed */
  uint64_t t_fail_ns;  /* %globaltimer when the rail stopped */
} nz_fault_record_t;

/* Launch status of a rail on this rank, written by its kernels into mapped
 * host memory (the engine's monitor reads it). Tags number
 * the rail's op entries (one per nz_rail_allreduce call / engine op). */
typedef struct {
  uint32_t ok_tag;      /* last entry whose every launch succeeded on this rank */
  uint32_t prog_tag;    /* entry of prog_chunk */
  uint64_t prog_chunk;  /* chunks [chunk_begin, prog_chunk) of that entry done on this rank */
  uint32_t start_tag;   /* last launch that started on the device */
  uint32_t fail_tag;    /* entry in which an injected dead link stopped this rank */
  uint64_t t_start_ns;  /* %globaltimer of that start */
  uint64_t t_fail_ns;   /* %globaltimer of that stop */
  uint32_t det_tag;     /* entry whose cross-rank wait timed out / was aborted here */
  uint32_t abort;       /* host -> device: stop waiting on peers (rail declared Failed) */
  uint64_t t_det_ns;    /* %globaltimer of that detection */
  uint32_t run_tag;     /* entry whose launch passed its start barrier (every rank arrived) */
  uint32_t reserved;
  uint64_t t_run_ns;    /* %globaltimer of that pass */
} nz_rail_status_t;
int nz_rail_status(const nz_rail_t* rail, nz_rail_status_t* out);
/* Unplanned failure injection: THIS rank's link of the rail
 * dies at `chunk` of its next nz_rail_allreduce — its kernels arrive at the
 * start barrier of the launch that covers that chunk and stop there, posting
 * nothing to the peers, and every later launch on this rank exits at once.
 * Peers are not told: their end-barrier waits time out (nz_rail_set_detect_us)
 * and their launches fail too. nz_rail_revive (on every rank) clears it. */
int nz_rail_inject_stall(nz_rail_t* rail, uint64_t chunk);
int nz_rail_revive(nz_rail_t* rail);
/* End-barrier budget of the rail's launches (failure detection), microseconds;
 * 0 restores the default (NEZHA_DETECT_US, else max(2000, 2 x range / 100 GB/s)). */
int nz_rail_set_detect_us(nz_rail_t* rail, double us);

/* Loopback rails: time every cross-rank grid on the stream it runs on (CUDA
 * events around each launch), and read + reset the totals (synchronizes). */
int nz_rail_loop_timing(nz_rail_t* rail, int enable);
int nz_rail_loop_time(nz_rail_t* rail, uint64_t* launches, double* total_us);

/* Non-blocking read of the rail's mapped fault word; clears it when `consume`. */
int nz_rail_poll_fault(nz_rail_t* rail, nz_fault_record_t* rec, int consume);
/* Device watchdog status: 0 ok, else a barrier timed out (the kernel bailed
 * out instead of hanging). Cleared by reading. */
int nz_rail_watchdog(nz_rail_t* rail);

/* --------------------------------------------------------------- engine --- */
typedef struct {
  int num_rails;             /* 1..3 */
  int kinds[3];              /* nz_rail_kind_t per rail, rail_id = index */
  int sm_budget[3];          /* CTA cap per rail (0 = all SMs) */
  int algorithm;             /* nz_algorithm_t, default RingChunked */
  double tau;                /* Eq. 3 gate, default 5 */
  double eta;                /* Eq. 7 step, default 0.05 */
  double convergence_eps;    /* default 0.01 */
  double sync_overhead_us;   /* < 0: measure at startup */
  int window;                /* Timer window, default 100 */
  int max_iters;             /* default 100 */
  int demote_after;          /* DESIGN.md P12; 0 disables */
  const char* rails_toml;    /* optional rails config text; NULL: calibrate */
  int calibrate_iters;       /* ops per size during startup calibration */
  uint64_t calibrate_max_bytes; /* largest calibrated size (default 1 GiB) */
  int timer_lag;             /* op k is sampled when op k + lag is issued (default 2) */
  int compute_pool;          /* SM arbitration of concurrent rails (P14):
                                0 off (default), 1 block (SPEC ComputePool), 2 shrink */
  int pool_tokens;           /* ComputePool total_tokens; 0 = the GPU's SM count */
  int tune_budgets;          /* 1: measure the NVLS / SM rails' CTA budgets and protocol
                                crossovers at startup (default 0 until validated) */
  int graph_safe;            /* 1: rails created with NZ_RAIL_FLAG_GRAPH_SAFE, so engine
                                allreduces can be captured in CUDA graphs (captured
                                ops are not Timer samples and are not monitored) */
  int monitor;               /* 1 (default): failure monitor thread + stream gates
                                (DESIGN.md §6b); 0: none (a failed rail raises at
                                nz_engine_synchronize) */
  double detect_us;          /* end-barrier budget floor; <= 0: default */
  double heartbeat_us;       /* monitor heartbeat interval, default 50000 */
  double readmit_hold_us;    /* healthy probes needed before readmit, default 1e6 */
} nz_engine_config_t;

void nz_engine_config_default(nz_engine_config_t* cfg);
/* Collective. Builds rails, measures profiles (unless rails_toml is given)
 * and sync overhead, and initialises the allocation table. */
int nz_engine_create(nz_comm_t* comm, const nz_engine_config_t* cfg, nz_engine_t** out);
int nz_engine_destroy(nz_engine_t* eng);

/* In-memory multi-rail allreduce of `bytes` bytes at offset 0 of the
 * symmetric buffers. `stream` (NULL = legacy default; on a loopback rank the
 * rank's own engine stream, since virtual ranks share the legacy stream) is
 * the caller's: the rails fork from it and join back into it, and with the
 * monitor on it passes each rail's part only through that rail's gate word
 * (DESIGN.md §6b). Asynchronous. */
int nz_engine_allreduce(nz_engine_t* eng, nz_buf_t* in, nz_buf_t* out, uint64_t bytes, int dtype, void* stream);
/* End to end from host memory (pinned or pageable): H2D into the engine's
 * UnboundBuffer, multi-rail allreduce, D2H into host_out, pipelined over
 * pieces. Synchronous. */
int nz_engine_allreduce_host(nz_engine_t* eng, const void* host_in, void* host_out, uint64_t bytes, int dtype);
/* Same pipeline for device memory the caller owns (not symmetric), e.g. a
 * PyTorch gradient bucket: staged through the engine's UnboundBuffer in
 * pieces, asynchronous on `stream` (NULL = legacy default); src == dst is
 * allowed. */
int nz_engine_allreduce_device(nz_engine_t* eng, const void* src, void* dst, uint64_t bytes, int dtype, void* stream);
/* Unplanned failure: THIS rank's link of `rail_id` dies at `chunk` of op
 * `op_seq` (nz_rail_inject_stall semantics). Call it on one rank only: the
 * others are not told and must detect it; every rank's monitor then agrees on
 * the orphan (min over ranks of completed chunks) and reroutes it (P9/P10). */
int nz_engine_inject_failure(nz_engine_t* eng, uint32_t op_seq, int rail_id, uint64_t chunk);
/* Readmits a previously failed rail: collective; probes the
 * rail until it has been healthy for readmit_hold_us, then re-enters it at
 * its last converged split. */
int nz_engine_readmit(nz_engine_t* eng, int rail_id);
int nz_engine_synchronize(nz_engine_t* eng);
uint32_t nz_engine_op_seq(const nz_engine_t* eng);
/* The engine's rail with this id (owned by the engine; NULL if none). */
nz_rail_t* nz_engine_rail(nz_engine_t* eng, int rail_id);

typedef struct {
  uint32_t op_seq;
  int failed_rail;
  int target_rail;
  uint64_t orphan_offset;
  uint64_t orphan_length;
  double detect_us;   /* device fault stamp -> host monitor saw it */
  double resume_us;   /* device fault stamp -> survivor started the orphan */
  double done_us;     /* device fault stamp -> orphan complete */
  double host_detect_us; /* device fault stamp -> this rank's monitor saw the failure
                            (host clock mapped onto %globaltimer, +-~2 us) */
  double device_detect_us; /* device fault stamp -> this rank's kernel gave up waiting
                              (0 on the rank whose link died) */
  double resume_after_detect_us; /* monitor saw the failure -> survivor started the orphan */
  uint64_t orphan_chunk;  /* first chunk rerouted = min over ranks of completed chunks */
  int stalled_here;       /* 1 on the rank whose link died */
} nz_failover_report_t;
/* Last completed failover (returns NZ_ERR_INVALID when none happened).
 * `t_fail` is the dead rank's device stamp, shared by the agreement. */
int nz_engine_last_failover(nz_engine_t* eng, nz_failover_report_t* rep);
/* Every failover so far, in order: count, and the i-th report. */
int nz_engine_failover_count(nz_engine_t* eng);
int nz_engine_failover_get(nz_engine_t* eng, int i, nz_failover_report_t* rep);

/* Warm restart: the allocation table, calibrated profiles and
 * sync overhead as JSON; load it on every rank (same text) to skip
 * re-convergence. */
int nz_engine_save_state(nz_engine_t* eng, char* out, size_t cap);
int nz_engine_load_state(nz_engine_t* eng, const char* json);

/* Timer totals per rail since the last reset (harvested ops only; call
 * nz_engine_synchronize first to harvest everything): ops, summed rail time
 * (fork -> rail done, us) and summed segment bytes. */
int nz_engine_rail_stats(nz_engine_t* eng, int rail_id, uint64_t* ops, double* total_us, uint64_t* total_bytes);
int nz_engine_stats_reset(nz_engine_t* eng);
/* Number of this library's kernels launched by this process so far. */
uint64_t nz_kernel_launch_count(void);

/* JSON snapshots: allocation table + profiles + health, and the plan the
 * engine would use for `bytes` (segments per rail). */
int nz_engine_state_json(nz_engine_t* eng, char* out, size_t cap);
int nz_engine_plan_json(nz_engine_t* eng, uint64_t bytes, char* out, size_t cap);
/* The plans (one per 256 MiB piece above 1 GiB) the last allreduce call ran,
 * with each segment's chunk size: what a checker needs to recompute it. */
int nz_engine_last_plan_json(nz_engine_t* eng, char* out, size_t cap);

/* -------------------------------------------------------------- planner --- */
/* Runs the balancer + fault logic over a scenario (rails, config, op stream,
 * injected latency model, failures; format in DESIGN.md §5) with no GPU, and
 * writes the decision log (one JSON object per line). Bit-exact contract with
 * oracle/planner.py. */
int nz_planner_run_trace(const char* scenario, char* out, size_t cap);

/* The planner driven op by op: the engine's nezha::Balancer with the rails
 * and profiles of a rails TOML (every rail needs a profile). The
 * engine's multi-rank flush agreement is the caller's `agree` callback: it
 * receives this rank's per-rail window means (in rail_id order) and must
 * replace them in place with the values every rank applies (the engine uses
 * the max over ranks); return 0 on success. Without a callback, identity. */
typedef struct nz_balancer nz_balancer_t;
typedef int (*nz_agree_fn)(void* ctx, int bucket, int n, const int* rail_ids, double* means);
int nz_balancer_create(const char* rails_toml, double tau, double eta, double sync_overhead_us, int window,
                       int demote_after, nz_balancer_t** out);
int nz_balancer_destroy(nz_balancer_t* b);
int nz_balancer_set_agreement(nz_balancer_t* b, nz_agree_fn fn, void* ctx);
/* Plans one op of `bytes` (JSON as in the planner trace) and keeps it
 * pending until nz_balancer_record reports its per-rail latencies. */
int nz_balancer_allocate(nz_balancer_t* b, uint64_t bytes, char* plan_json, size_t cap);
int nz_balancer_record(nz_balancer_t* b, int n, const int* rail_ids, const double* us, int* flushed);
int nz_balancer_table_json(nz_balancer_t* b, char* out, size_t cap);

/* ------------------------------------------------------------ emulation --- */
/* Single-GPU emulation of one rank of the SM rail (ndst == world: fold and
 * store to every rank's output) or of the CE rail's local reduce (ndst == 1)
 * over [lo, hi) with the segment's order geometry. All `world` input and
 * output buffers live on the current device; no barriers are issued, so the
 * caller runs the virtual ranks one after another. Lets the exact rail
 * kernels be parity-tested for N = 2..8 on a single B200. grid <= 0: auto. */
int nz_emulate_fold(int world, int rank, int dtype, const void* const* src, void* const* dst, int ndst,
                    uint64_t seg_off, uint64_t seg_len, uint64_t chunk_bytes, uint64_t lo, uint64_t hi, int grid,
                    void* stream);


/* ----------------------------------------------------------------- pool --- */
/* Host ComputePool with the semantics pinned in include/nezha/compute_pool.hpp.
 * phase: 0 io, 1 communication, 2 computation. nz_pool_acquire blocks when
 * `blocking`, else sets *grant = -1 when it would block. */
typedef struct nz_pool nz_pool_t;
int nz_pool_create(int total_tokens, nz_pool_t** out);
int nz_pool_destroy(nz_pool_t* pool);
int nz_pool_declare(nz_pool_t* pool, int rail_id, int io, int communication, int computation);
int nz_pool_acquire(nz_pool_t* pool, int rail_id, int phase, int blocking, int* grant);
int nz_pool_release(nz_pool_t* pool, int rail_id, int phase);
/* Computation tokens outstanding, or a negative error code. */
int nz_pool_outstanding(const nz_pool_t* pool);
int nz_pool_waiting(const nz_pool_t* pool);
/* The engine's stream-order arbitration of one op (planComputeGrants):
 * mode 0 off, 1 block (SPEC), 2 shrink. For each of the n rails (in order)
 * writes its grant and a bitmask of the rail ids (< 32) it waits for. */
int nz_pool_plan(int total_tokens, int mode, int n, const int* rail_ids, const int* demands, int* grants,
                 uint32_t* wait_masks);

/* ----------------------------------------------------------------- core --- */
uint64_t nz_core_ring_volume(int node_count, uint64_t payload);
int nz_core_bucket_of(uint64_t size);
uint64_t nz_core_default_chunk_bytes(uint64_t seg_len, int world, int algorithm);
/* calibrate(samples) -> CalibratedProfile (P15):
 * *interpolated = 1 when the samples had to become an interpolation table. */
int nz_core_calibrate(const uint64_t* sizes, const double* lat_us, int n, double* t_setup_us, double* bandwidth_bps,
                      int* interpolated, double* max_rel_residual);

#ifdef __cplusplus
}
#endif

#endif /* NEZHA_B200_H */
