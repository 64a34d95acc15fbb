/*
 * rkr.h -- C ABI of the B200-native rk-Rotor chain solver (librkr.so).
 *
 * This is the drop-in boundary for the hot path named by BASELINE.json's
 * north_star: the rk-Rotor chain dynamic program of
 * /root/reference/proj/include/remat/chain_dp.hpp.  The reference has no FFI
 * layer of its own (its "operator API" is the header-only C++ API in
 * namespace remat), so every entry point below cites the C++ interface it
 * replaces; include/remat_b200/chain_dp.hpp re-exposes that exact C++ API on
 * top of these calls.
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross the ABI.  Every call
 *    returns an rkr_status; rkr_last_error() gives a thread-local message.
 *  - Host buffers are caller-owned.  rkr_table owns its device memory.
 *  - The DP runs on the GPU only.  There is no CPU fallback: on a host
 *    without a usable sm_100 device every compute call returns RKR_ERR_CUDA.
 *  - A table handle is immutable after creation; distinct handles may be
 *    used from distinct threads.
 */
#ifndef RKR_H
#define RKR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RKR_ABI_VERSION 2

/* Mirrors remat::kInfTime (chain_dp.hpp:23). */
#define RKR_INF_TIME ((int64_t)(INT64_MAX / 4))

typedef enum {
    RKR_OK = 0,
    RKR_ERR_INVALID = 1,     /* remat::ValidationError (chain_dp.hpp:33,58,84,94,203) */
    RKR_ERR_INFEASIBLE = 2,  /* remat::InfeasibleBudget (chain_dp.hpp:214,245,261,285) */
    RKR_ERR_CUDA = 3,        /* device missing / launch or copy failure */
    RKR_ERR_OOM = 4,         /* device allocation failed */
    RKR_ERR_CAPACITY = 5,    /* caller's output buffer too small (size reported) */
    RKR_ERR_ARGUMENT = 6     /* null pointer / index out of range */
} rkr_status;

/* DpArg::Kind (chain_dp.hpp:44-47). */
typedef enum { RKR_ARG_NONE = 0, RKR_ARG_OPTION = 1, RKR_ARG_CUT = 2 } rkr_arg_kind;

/* ScheduleOp::Kind (types.hpp:346-362).  COMPUTE is the loss op of block
 * L-1; FORGET drops block j's input activation. */
typedef enum {
    RKR_OP_COMPUTE = 0,
    RKR_OP_FORGET = 1,
    RKR_OP_BLOCK_FWD = 2,
    RKR_OP_BLOCK_BWD = 3
} rkr_op_kind;

typedef struct {
    int32_t kind;   /* rkr_op_kind */
    int32_t block;
    int32_t option; /* option id for BLOCK_FWD/BLOCK_BWD, -1 otherwise */
} rkr_op;

/* remat::OptionMenu (chain_dp.hpp:16-21) flattened: options of block i are
 * entries [option_offsets[i], option_offsets[i+1]) in menu order; the fields
 * are remat::BlockOption's (types.hpp:330-344); has_bwd[o] says whether the
 * optional time_bwd is present.  act_sizes holds a_0..a_L in bytes. */
typedef struct {
    int32_t n_blocks;
    const int32_t* option_offsets; /* [n_blocks + 1] */
    const int32_t* option_id;
    const int64_t* time_fwd;
    const int64_t* time_bwd;
    const uint8_t* has_bwd;
    const int64_t* save_mem;
    const int64_t* peak_fwd;
    const int64_t* peak_fwd_pre;
    const int64_t* peak_bwd;
    const int64_t* act_sizes;      /* [n_blocks + 1] */
} rkr_menu;

typedef enum {
    RKR_WIDTH_AUTO = 0, /* 32-bit costs when the host overflow proof holds, else 64 */
    RKR_WIDTH_64 = 64   /* force the general int64 kernels */
} rkr_width;

typedef enum {
    RKR_KERNEL_PERSISTENT = 0, /* one persistent launch per fill (default): budget tiles
                                  when they fit one CTA per SM, else the work queue */
    RKR_KERNEL_DIAGONAL = 1,   /* one launch per anti-diagonal (the simple wavefront) */
    RKR_KERNEL_QUEUE = 2,      /* persistent, dataflow-queue scheduled (row-segment items) */
    RKR_KERNEL_TILES = 3       /* persistent, one CTA per budget tile (RKR_ERR_INVALID if
                                  the table does not fit) */
} rkr_kernel;

/* Kernel tuning overrides (rkr_exec.tune bits).  0 = the library's measured
 * choices; the bits exist for A/B measurements and for
 * tests that pin one variant.  Results are identical under every setting. */
typedef enum {
    RKR_TUNE_NO_TILES = 1 << 0,    /* never the budget-tile kernel (K1t) */
    RKR_TUNE_JOBS = 1 << 1,        /* K1t as tile jobs even when its tiles fit one CTA per SM */
    RKR_TUNE_COMM_OFF = 1 << 2,    /* K1t without the communication warp */
    RKR_TUNE_COMM_ON = 1 << 3,     /* K1t with the communication warp */
    RKR_TUNE_SPLIT_OFF = 1 << 4,   /* no split tails on late diagonals */
    RKR_TUNE_SPLIT_ON = 1 << 5,    /* split tails (with the communication warp) */
    RKR_TUNE_STREAM = 1 << 6,      /* streamed cut programs even when they fit shared memory */
    RKR_TUNE_BATCH_QUEUE = 1 << 7, /* batches on the row-segment queue (K1p) */
    RKR_TUNE_PROFILE = 1 << 8,     /* host phase timers on stderr (synchronises: never for timing) */
    RKR_TUNE_WIDE_SEARCH = 1 << 9, /* min-feasible search by filling the wide table (as the
                                      reference does) instead of the threshold recurrence */
    RKR_TUNE_UNIFORM = 1 << 10,    /* tile jobs all of one width (no half tiles in the last wave) */
    RKR_TUNE_MIXED = 1 << 11,      /* (tests) tile jobs: half 32-slot, half 16-slot tiles */
    RKR_TUNE_NO_PRUNE = 1 << 12    /* K1t: scan every option of open rows (no dominance pruning) */
} rkr_tune;

/* Execution settings; pass NULL for defaults (device 0, the library's shared
 * per-device stream, auto width, persistent kernel, measured tuning). */
typedef struct {
    int32_t device;
    void* stream;       /* cudaStream_t, or NULL for the library's per-device stream */
    int32_t width;      /* rkr_width */
    int32_t kernel;     /* rkr_kernel */
    int32_t tune;       /* rkr_tune bits, 0 = defaults */
    int32_t tile_rows;  /* K1t rows per warp: 0 = auto, 1 (32-slot tiles) or 2 (16-slot tiles) */
    int32_t reserved[2];
} rkr_exec;

typedef struct rkr_table rkr_table;

const char* rkr_last_error(void);
int32_t rkr_abi_version(void);
/* 1 when an sm_100 device is visible and the kernels can run here. */
int32_t rkr_device_ok(int32_t device);

/* remat::quantize (chain_dp.hpp:32-39) and remat::to_units (:41). */
rkr_status rkr_quantize(int64_t budget_bytes, int32_t units, int64_t* unit,
                        int64_t* budget_units);
int64_t rkr_to_units(int64_t bytes, int64_t unit);

/* remat::DpTable::DpTable(menu, unit, m_max) (chain_dp.hpp:56-101): validates
 * the menu, does the per-block unit precompute on the host, copies it to the
 * device and fills every cell (s <= t, 0 <= m <= m_max) with the wavefront
 * kernels.  Returns when the fill has been enqueued on the handle's stream. */
rkr_status rkr_table_create(const rkr_menu* menu, int64_t unit, int32_t m_max,
                            const rkr_exec* exec, rkr_table** out);
void rkr_table_destroy(rkr_table* table);

/* DpTable::length/unit/m_max/act_units (chain_dp.hpp:113-116). */
int32_t rkr_table_length(const rkr_table* table);
int64_t rkr_table_unit(const rkr_table* table);
int32_t rkr_table_m_max(const rkr_table* table);
int64_t rkr_table_act_units(const rkr_table* table, int32_t i);
/* 32 or 64: the cost width the fill ran in (bookkeeping only; every value
 * leaving the library is int64 and bit-exact). */
int32_t rkr_table_width(const rkr_table* table);
/* The fill kernel the table runs: RKR_KERNEL_TILES, RKR_KERNEL_QUEUE or
 * RKR_KERNEL_DIAGONAL (RKR_KERNEL_PERSISTENT resolves to one of the first two). */
int32_t rkr_table_kernel(const rkr_table* table);
/* DpTable::max_candidates_per_cell / worst_cell_allowance (:118-120),
 * computed in closed form from the menu (the device fill visits exactly the
 * reference's candidate sequence). */
rkr_status rkr_table_work_bound(const rkr_table* table, int64_t* max_candidates_per_cell,
                                int64_t* worst_cell_allowance);

/* DpTable::opt / arg (chain_dp.hpp:103-112): m < 0 -> RKR_INF_TIME / NONE,
 * m > m_max clamps to m_max.  Requires 0 <= s <= t < L. */
rkr_status rkr_table_opt(const rkr_table* table, int32_t s, int32_t t, int32_t m, int64_t* out);
rkr_status rkr_table_arg(const rkr_table* table, int32_t s, int32_t t, int32_t m,
                         int32_t* kind, int32_t* value);

/* Bulk copy of one row (s, t), m = 0..m_max, as the reference stores it:
 * opt int64, arg kind and value.  Any output pointer may be NULL. */
rkr_status rkr_table_row(const rkr_table* table, int32_t s, int32_t t, int64_t* opt,
                         int8_t* kind, int32_t* value);
/* Bulk copy of the whole table, rows in s-major upper-triangular order
 * (row(s,t) = s*L - s*(s-1)/2 + (t-s)), each m_max+1 long. */
rkr_status rkr_table_download(const rkr_table* table, int64_t* opt, int8_t* kind,
                              int32_t* value);

/* remat::build_schedule_rec(table, menu, chain, s, t, m, out)
 * (chain_dp.hpp:211-246), run on the device; only the ops return.  On
 * RKR_ERR_CAPACITY *n_ops holds the required count.  On RKR_ERR_INFEASIBLE
 * *n_ops holds the ops emitted before the infeasible cell (as the
 * reference's out-vector would). */
rkr_status rkr_backtrack(const rkr_table* table, int32_t s, int32_t t, int32_t m, rkr_op* ops,
                         int64_t cap, int64_t* n_ops);

/* build_schedule_rec with the CALLER's menu, as the reference does: the
 * option decided at a cell is looked up by id in `menu` (first match,
 * chain_dp.hpp:200-205) and its pack shift to_units(save_mem - act_sizes[s])
 * taken from there (:228); cut shifts come from the table (:240).  A menu
 * lacking the option: RKR_ERR_INVALID ("menu for block s lacks option id",
 * the reference's ValidationError), *n_ops = the ops emitted before it.
 * menu == NULL or the table's own menu: the same as rkr_backtrack. */
rkr_status rkr_backtrack_menu(const rkr_table* table, const rkr_menu* menu, int32_t s, int32_t t,
                              int32_t m, rkr_op* ops, int64_t cap, int64_t* n_ops);

/* The same walk split in two: _async enqueues it on the table's stream (no
 * host sync), _fetch waits and copies the ops (same statuses as above). */
rkr_status rkr_backtrack_async(rkr_table* table, int32_t s, int32_t t, int32_t m);
rkr_status rkr_backtrack_fetch(rkr_table* table, rkr_op* ops, int64_t cap, int64_t* n_ops);

/* First m with opt(s, t, m) < inf, or -1 (the scan in solve_chain's
 * infeasible branch, chain_dp.hpp:280-284), computed on the device. */
rkr_status rkr_first_feasible(const rkr_table* table, int32_t s, int32_t t, int32_t* m_out);

/* remat::solve_chain(chain, menu, budget_bytes, units) (chain_dp.hpp:255-296)
 * in one call: quantize, fill, top cell, device backtrack; on infeasibility
 * the wide-table min-feasible search, returned in *min_feasible (bytes, or -1)
 * with RKR_ERR_INFEASIBLE. */
rkr_status rkr_solve_chain(const rkr_menu* menu, int64_t budget_bytes, int32_t units,
                           const rkr_exec* exec, rkr_op* ops, int64_t cap, int64_t* n_ops,
                           int64_t* opt_time, int64_t* unit, int32_t* m_top,
                           int64_t* min_feasible);

/* Wait for all work queued on the table's stream. */
rkr_status rkr_table_sync(const rkr_table* table);

/* Re-run the whole fill from the device-resident menu (no host work, async):
 * the device-only step bench.py times. */
rkr_status rkr_table_refill(rkr_table* table);
/* Refill, then walk build_schedule_rec from (s, t, m) on the device (async;
 * collect with rkr_backtrack_fetch).  With the budget-tile fill the walk is
 * fused into the fill launch: the last CTA to finish walks. */
rkr_status rkr_table_refill_walk(rkr_table* table, int32_t s, int32_t t, int32_t m);
/* The cudaStream_t every kernel of this table is launched on. */
void* rkr_table_stream(const rkr_table* table);
/* Bytes copied host->device by rkr_table_create (the staged menu precompute). */
int64_t rkr_table_h2d_bytes(const rkr_table* table);
/* Device bytes the table holds (menu, scratch, opt and arg rows). */
int64_t rkr_table_device_bytes(const rkr_table* table);

/* ---- Batches: many independent tables, ONE persistent fill launch ---------
 * (BASELINE config 4: budget sweeps x model instances.)  Table i is built
 * exactly as rkr_table_create(menus[i], units[i], m_max[i], exec) would build
 * it; all tables share one cost width (64 if any table needs it).
 * rkr_batch_table returns a borrowed handle with the whole per-table API
 * (opt/arg/row/download/backtrack/first_feasible); do not destroy it. */
typedef struct rkr_batch rkr_batch;
rkr_status rkr_batch_create(const rkr_menu* const* menus, const int64_t* units,
                            const int32_t* m_max, int32_t n, const rkr_exec* exec,
                            rkr_batch** out);
int32_t rkr_batch_size(const rkr_batch* batch);
rkr_table* rkr_batch_table(rkr_batch* batch, int32_t i);
rkr_status rkr_batch_refill(rkr_batch* batch);
void* rkr_batch_stream(const rkr_batch* batch);
rkr_status rkr_batch_sync(const rkr_batch* batch);
void rkr_batch_destroy(rkr_batch* batch);

/* remat::solve_chain for n budgets of one chain (the per-budget loop of the
 * reference's cmd_sweep, tools/remat.cpp:240-255), all tables in one batched
 * fill; top cells, schedules and the min-feasible search of infeasible
 * budgets are batched too.  Per budget i: status[i] is RKR_OK or
 * RKR_ERR_INFEASIBLE (min_feasible[i] then holds the threshold in bytes, or
 * -1); opt_time/unit/m_top as rkr_solve_chain.  Schedules are concatenated in
 * ops; budget i's ops are [ops_offsets[i], ops_offsets[i+1]).  If ops_cap is
 * too small, returns RKR_ERR_CAPACITY with ops_offsets[n] = ops needed (every
 * other output is valid).  Budgets are processed in the given order; sorting,
 * de-duplication and the monotonicity check (remat.cpp:232-263) are the
 * caller's (see the host sweep helpers). */
rkr_status rkr_sweep(const rkr_menu* menu, const int64_t* budgets, int32_t n, int32_t units,
                     const rkr_exec* exec, int32_t* status, int64_t* opt_time, int64_t* unit,
                     int32_t* m_top, int64_t* min_feasible, rkr_op* ops, int64_t ops_cap,
                     int64_t* ops_offsets);

/* rkr_sweep over several chains at once (cmd_sweep for each, remat.cpp:217-
 * 263, sharing one batch and one fill launch): chain c has n_budgets[c]
 * budgets, stored consecutively in `budgets` in chain order; every output is
 * indexed like `budgets` (total n = sum of n_budgets), with the results,
 * statuses and op layout of one rkr_sweep call per chain, concatenated. */
rkr_status rkr_sweep_chains(const rkr_menu* const* menus, const int32_t* n_budgets,
                            int32_t n_chains, const int64_t* budgets, int32_t units,
                            const rkr_exec* exec, int32_t* status, int64_t* opt_time,
                            int64_t* unit, int32_t* m_top, int64_t* min_feasible, rkr_op* ops,
                            int64_t ops_cap, int64_t* ops_offsets);

/* ---- Budget-axis sharding (BASELINE config 5) -----------------------------
 * One table split into n contiguous budget ranges ("shards"), shard i on
 * devices[i] (NULL: all on exec->device).  Each shard is filled by the
 * persistent kernel; an item whose slots are the next shard's halo (its
 * lowest `pad` slots read shifted columns of this shard) stores them straight
 * into the next shard's rows -- peer memory over NVLink when the shards live
 * on different GPUs -- and signals it with a counter, so the exchange is
 * fused into the fill (no collective call, no host round trip per diagonal).
 * Every shard must own at least `pad` slots.  Reads take GLOBAL budget slots;
 * results are bit-identical to the unsharded table. */
typedef struct rkr_sharded rkr_sharded;
rkr_status rkr_sharded_create(const rkr_menu* menu, int64_t unit, int32_t m_max, int32_t n_shards,
                              const int32_t* devices, const rkr_exec* exec, rkr_sharded** out);
int32_t rkr_sharded_count(const rkr_sharded* sharded);
rkr_status rkr_sharded_range(const rkr_sharded* sharded, int32_t shard, int32_t* m_lo,
                             int32_t* m_hi);
rkr_table* rkr_sharded_shard(rkr_sharded* sharded, int32_t shard);  /* borrowed, local slots */
rkr_status rkr_sharded_refill(rkr_sharded* sharded);
rkr_status rkr_sharded_sync(const rkr_sharded* sharded);
rkr_status rkr_sharded_opt(const rkr_sharded* sharded, int32_t s, int32_t t, int32_t m,
                           int64_t* out);
rkr_status rkr_sharded_row(const rkr_sharded* sharded, int32_t s, int32_t t, int64_t* opt,
                           int8_t* kind, int32_t* value);
rkr_status rkr_sharded_backtrack(rkr_sharded* sharded, int32_t s, int32_t t, int32_t m,
                                 rkr_op* ops, int64_t cap, int64_t* n_ops);
void rkr_sharded_destroy(rkr_sharded* sharded);

/* Multi-process budget sharding (one process per GPU, e.g. torchrun):
 * rank r calls rkr_shard_create(..., n_shards, r, ...) (same menu/unit/m_max on
 * every rank), exchanges rkr_shard_export's 64-byte CUDA IPC handle and 8
 * int64 info words with its neighbours (any host channel: torch.distributed,
 * MPI, files), links to shard r+1 with rkr_shard_link, then every fill is
 * rkr_shard_zero on all ranks -> a host barrier -> rkr_shard_launch on all
 * ranks.  The halo exchange happens inside the kernels over NVLink peer
 * memory.  rkr_shard_backtrack walks the whole table from shard 0's process
 * (handles/infos of all n shards, index 0 ignored); m is a global slot.
 * Shard tables are ordinary rkr_table handles for accessors (local slots,
 * rkr_shard_range gives [m_lo, m_hi)); destroy with rkr_table_destroy. */
rkr_status rkr_shard_create(const rkr_menu* menu, int64_t unit, int32_t m_max, int32_t n_shards,
                            int32_t shard, const rkr_exec* exec, rkr_table** out);
rkr_status rkr_shard_range(const rkr_table* shard, int32_t* m_lo, int32_t* m_hi);
rkr_status rkr_shard_export(const rkr_table* shard, void* ipc_handle, int64_t* info);
rkr_status rkr_shard_link(rkr_table* shard, const void* next_ipc_handle, const int64_t* next_info);
rkr_status rkr_shard_zero(rkr_table* shard);
rkr_status rkr_shard_launch(rkr_table* shard);
/* The walk mirror (optional, before the fill): shard 0 allocates a full-width
 * copy of the arg table (m_max = the table's global m_max) and exports it;
 * every other shard attaches it, and from then on each fill also stores its
 * codes there (peer stores), so rkr_shard_backtrack on shard 0 reads only
 * local memory instead of one NVLink round trip per hop.  info: 8 int64. */
rkr_status rkr_shard_mirror(rkr_table* shard0, int32_t m_max, void* ipc_handle, int64_t* info);
rkr_status rkr_shard_attach_mirror(rkr_table* shard, const void* ipc_handle, const int64_t* info);
rkr_status rkr_shard_backtrack(rkr_table* shard0, int32_t n_shards, const void* const* ipc_handles,
                               const int64_t* infos, int32_t s, int32_t t, int32_t m, rkr_op* ops,
                               int64_t cap, int64_t* n_ops);

/* Schedule validation gate (host, exact): replays ops in the chain-level
 * block-atomic memory model the DP optimises (the model of the reference's
 * tests/test_helpers.hpp:249-322) and returns the makespan and the peak in
 * bytes.  A malformed schedule gives RKR_ERR_INVALID and *bad_op = index. */
rkr_status rkr_replay(const rkr_menu* menu, const rkr_op* ops, int64_t n_ops, int64_t* peak,
                      int64_t* makespan, int64_t* bad_op);

/* Diagnostics (persistent kernel only): 6 globaltimer stamps per item of the
 * next fills {dequeued, diagonal k-2 met, bulk cuts done, diagonal k-1 met,
 * tail done, published}; item_k/item_j (nullable) receive each item's
 * diagonal and tile. */
rkr_status rkr_debug_trace(rkr_table* table, int32_t enable);
int64_t rkr_debug_trace_items(const rkr_table* table);
rkr_status rkr_debug_trace_read(const rkr_table* table, uint64_t* stamps, int32_t* item_k,
                                int32_t* item_j);

#ifdef __cplusplus
}
#endif

#endif /* RKR_H */
