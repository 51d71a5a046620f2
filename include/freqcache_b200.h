/*
 * freqcache_b200 — C ABI of the B200-native frequency-aware embedding cache.
 *
 * Drop-in boundary for the reference's cached-embedding path
 * (/root/reference/pkg/src/freqcache, a pure-Python/numpy package with no FFI of
 * its own). Each entry point replaces one reference call; the citation is the
 * reference function whose semantics it reproduces bit-for-bit. The Python host
 * package `paper_2208_05321_b200` binds these with ctypes and keeps the reference
 * names, argument meanings and exception classes.
 *
 * Conventions
 *  - Plain pointers and sizes only. "dev" pointers are CUDA device pointers,
 *    "host" pointers are host memory. Streams are cudaStream_t passed as void*.
 *  - Every call returns an fc_status (0 = OK). Validation errors are reported
 *    BEFORE any state mutation, like the reference (cache_manager.py:261-282).
 *  - Calls that must hand scalars back (prepare, flush, warmup) synchronise the
 *    given stream; everything else is stream-ordered and asynchronous.
 *  - One handle is single-writer; independent handles may run
 *    concurrently on different streams/devices.
 */
#ifndef FREQCACHE_B200_H
#define FREQCACHE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fc_status {
  FC_OK = 0,
  FC_ERR_BATCH_EXCEEDS_CAPACITY = 1, /* BatchExceedsCapacity   cache_manager.py:35-40,278-282 */
  FC_ERR_ID_OUT_OF_RANGE = 2,        /* ValueError("id out of range: ...")  :272-275 */
  FC_ERR_INSUFFICIENT_EVICTABLE = 3, /* InsufficientEvictable  :43-44,67-72 */
  FC_ERR_INSUFFICIENT_FREE_SLOTS = 4,/* InsufficientFreeSlots  :47-52,313-317 */
  FC_ERR_BUFFER_TOO_SMALL = 5,       /* BufferTooSmall         transmitter.py:28-29,85-88 */
  FC_ERR_CUDA = 6,
  FC_ERR_BAD_ARG = 7,                /* ValueError for bad modes / sizes */
  FC_ERR_SLOT_OUT_OF_RANGE = 8,      /* IndexError             cache_manager.py:397-399 */
  FC_ERR_NOT_EMPTY = 9,              /* ValueError("warmup requires an empty cache") :365-366 */
  FC_ERR_NO_SLOW_TIER = 10
} fc_status;

typedef enum fc_write_back { FC_WB_DIRTY_ONLY = 0, FC_WB_ALWAYS = 1 } fc_write_back;     /* :31 */
typedef enum fc_evict_mode { FC_EVICT_OCCUPANCY_AWARE = 0, FC_EVICT_PAPER_LITERAL = 1 } fc_evict_mode; /* :32 */
typedef enum fc_pool_mode { FC_POOL_SUM = 0, FC_POOL_MEAN = 1 } fc_pool_mode;
typedef enum fc_optim { FC_OPT_SGD = 0, FC_OPT_ADAGRAD = 1 } fc_optim;

typedef struct fc_cache fc_cache;   /* opaque handle: one CacheStack (cache_manager.py:441-562) */

/* Outcome of one prepare call (PrepareResult, cache_manager.py:173-194, plus the
 * two TransferReports' row counts, transmitter.py:62-72). */
typedef struct fc_prepare_info {
  int64_t unique;        /* |U| */
  int64_t hits;
  int64_t misses;        /* rows admitted slow -> fast */
  int64_t evictions;     /* victims chosen */
  int64_t rows_to_slow;  /* victims written back (dirty_only filters by dirty bit) */
  int64_t free_count;    /* free slots after the call */
  int64_t bad_id;        /* offending id for FC_ERR_ID_OUT_OF_RANGE */
  int64_t candidates;    /* evictable rows seen when eviction ran (diagnostic) */
} fc_prepare_info;

/* Device pointers of the handle-owned state, for zero-copy views (torch tensors). */
typedef struct fc_views {
  float* fast_rows;       /* [capacity, row_width] fp32 fast tier (FastTierStore.slots)  */
  int32_t* slot_to_rank;  /* [capacity]   (CacheState.slot_to_rank, int64 in reference)  */
  int32_t* rank_to_slot;  /* [num_ids]    (CacheState.rank_to_slot)                      */
  uint8_t* dirty;         /* [capacity]   (CacheState.dirty)                             */
  int32_t* rank_of;       /* [num_ids]    (IdxMap.rank_of on device)                     */
  float* fast_state;      /* [capacity, state_width] optimizer state or NULL             */
  int64_t capacity, num_ids, dim, state_width;
} fc_views;

/* ---- lifecycle ------------------------------------------------------------ */
/* CacheState(capacity, num_ids) + FastTierStore + Transmitter(buffer_bytes)
 * (cache_manager.py:129-139, store.py:62-87, transmitter.py:75-94).
 * state_width: optimizer-state columns cached with each row (0 = none,
 * dim = element-wise Adagrad). buffer_bytes only drives message accounting and
 * the staged engine's chunk size (chunk = floor(buffer/row_bytes) rows). */
int fc_create(int64_t num_ids, int64_t capacity, int32_t dim, int32_t state_width,
              int32_t write_back, int32_t evict_mode, int64_t buffer_bytes, int32_t device,
              fc_cache** out);
int fc_destroy(fc_cache* h);
const char* fc_last_error(void);
int fc_get_views(fc_cache* h, fc_views* out);

/* Pinned, device-mapped host memory for the slow tier (page-locked once). */
int fc_host_alloc(int64_t bytes, void** out);
int fc_host_free(void* p);

/* IdxMap.rank_of (freq_stats.py:52-73), host int64[num_ids] -> device int32. */
int fc_set_idx_map(fc_cache* h, const int64_t* rank_of_host, void* stream);

/* SlowTierStore (store.py:39-59): rank-indexed rows [num_ids, dim] (+ optional
 * state rows [num_ids, state_width]) in pinned mapped host memory from
 * fc_host_alloc (or any cudaHostRegister-ed range). Row strides in floats. */
int fc_attach_slow_tier(fc_cache* h, float* rows_host, int64_t row_stride,
                        float* state_host, int64_t state_stride);

/* Per-call modes of prepare_cache (write_back, evict_mode kwargs, cache_manager.py:241-245).
 * Changing them while a prefetch is outstanding is refused; re-setting the same modes is not. */
int fc_set_modes(fc_cache* h, int32_t write_back, int32_t evict_mode);
/* The staging buffer of the transmitter passed to prepare_cache (transmitter.py:75-94; the
 * reference takes the transmitter per call). Only BufferTooSmall and the message accounting
 * depend on it. Refused while a prefetch is outstanding (unless unchanged). */
int fc_set_buffer_bytes(fc_cache* h, int64_t buffer_bytes);
/* CacheState.free_count after the last synchronising call. */
int64_t fc_free_count(fc_cache* h);

/* Transfer engine. 0 (default): one kernel pairs each staged victim write-back
 * (HBM -> pinned slow tier) with an admission (slow tier -> slot), all SM-issued
 * over the host link; the slow tier is current when prepare returns.
 * 1: victims are staged in HBM (double-buffered) and shipped D2H by the copy
 * engine on a side stream, then scattered into the slow tier by host threads,
 * overlapped with later work; admissions read the newest copy (HBM stage if the
 * rank is still pending). The slow tier is current after fc_flush / fc_drain. */
int fc_set_engine(fc_cache* h, int32_t engine);
int fc_drain(fc_cache* h);
/* fc_drain as a stream-ordered wait: work queued on `stream` after this call runs once every
 * write-back queued so far has landed in the slow tier; the host does not block. */
int fc_drain_stream(fc_cache* h, void* stream);

/* Measurement hook (no reference counterpart): with enable=1 every prepare records
 * CUDA events around the whole call and around the host-link transfer kernel.
 * out (returned, then reset): [0] sum prepare ms, [1] sum transfer-kernel ms, [2] calls,
 * [3] bytes the transfer kernel moved over the host link (4*(dim+state)*(admitted +
 * written-back rows) for engine 0, admitted rows only for engine 1), [4] victim bytes
 * (upper bound of the write-back), [5] host ms spent waiting for async write-backs,
 * [6] host scatter ms and [7] scatter jobs completed (engine 1), [8] transfer launches
 * timed (prefetch pipeline: [1] covers k_admit_stage), [9] rows written back to the slow
 * tier and [10] bytes shipped device -> host for them (engine 1, exact), [11] host scatter
 * threads (engine 1; bound to the GPU's local CPUs). `out` holds 12 doubles. */
int fc_profile(fc_cache* h, int32_t enable, double* out);

/* Timeline tracing (diagnostics, no reference counterpart): while enabled the
 * pipeline records tagged CUDA events (1/2 index phase begin/end, 3/4 miss staging
 * begin/end, 5/6 commit begin/end) and fc_trace_mark adds caller tags on any
 * stream. fc_trace_read returns up to `max` (tag, ms since the first event) pairs. */
int fc_trace(fc_cache* h, int32_t enable);
int fc_trace_mark(fc_cache* h, int32_t tag, void* stream);
int64_t fc_trace_read(fc_cache* h, int32_t* tags, double* ms, int64_t max);

/* ---- the cache verbs ------------------------------------------------------- */
/* warmup (cache_manager.py:351-390): ranks 0..k-1 -> slots 0..k-1; empty cache only. */
int fc_warmup(fc_cache* h, int64_t k, void* stream);

/* prepare_cache (cache_manager.py:234-348), the per-batch hot path.
 * ids_dev: n ids (int64 if ids_bytes==8, int32 if 4). Outputs (device, caller
 * allocated, capacity >= min(n, capacity) entries; `inverse` n entries):
 * unique ids ascending, their counts, ranks and final slots, and for every id
 * its position in the unique list (PrepareResult.slots_for_ids, :187-190).
 * Synchronises `stream`; fills `info`. On error nothing was mutated. */
int fc_prepare(fc_cache* h, const void* ids_dev, int32_t ids_bytes, int64_t n, int64_t batch_seq,
               int32_t* unique_ids, int32_t* unique_counts, int32_t* unique_ranks,
               int32_t* unique_slots, int32_t* inverse, void* stream, fc_prepare_info* info);

/* Prefetch pipeline (extension; the paper's future-work prefetch).
 * fc_prepare_begin launches batch t+1's prepare without waiting for batch t's
 * forward/backward: the index phase (dedup, lookups, victim and slot choice, every
 * slot-table change; no row and no dirty bit touched) runs on `stream`, and the
 * admitted rows are staged host -> HBM on a library-owned transfer stream. Outputs
 * are as fc_prepare's and become valid once fc_prepare_commit returns.
 * fc_prepare_commit, on the stream that runs the forward/backward, writes the
 * victims (already carrying batch t's update) to the write-back stage and moves the
 * staged rows into their slots; it fills `info` (rows_to_slow = -1: the dirty filter
 * runs on device) and reports validation errors (nothing is mutated on error).
 * The resulting cache state, slot assignment and write-backs are bit-identical to
 * calling fc_prepare at commit time. Requires the async engine (fc_set_engine 1).
 * Up to two begins may be outstanding (commits are FIFO): fc_prepare_begin(t+1)
 * before fc_prepare_commit(t) lets batch t+1's index phase start on the device as
 * soon as batch t's ends (its staging is then launched by commit(t); not with
 * FC_XFER_AFTER_UPDATE). The synchronous verbs refuse while any is outstanding. */
int fc_prepare_begin(fc_cache* h, const void* ids_dev, int32_t ids_bytes, int64_t n, int64_t batch_seq,
                     int32_t* unique_ids, int32_t* unique_counts, int32_t* unique_ranks, int32_t* unique_slots,
                     int32_t* inverse, void* stream);
int fc_prepare_commit(fc_cache* h, void* stream, fc_prepare_info* info);
/* Rows the last fc_prepare_commit wrote back (its dirty filter ran on device);
 * waits for that commit's kernels. 0 after a synchronous fc_prepare. */
int fc_last_writebacks(fc_cache* h, int64_t* rows);

/* Memory report (replaces CacheStack.memory_report, cache_manager.py:553-562, which counts
 * fast rows + the 64 MiB TransferBuffer + index arrays): every device allocation the
 * cache holds, by category, so the total matches the device memory it takes. The staging
 * buffers start at buffer_bytes worth of rows and grow only when a batch needs more. The
 * cache's fixed arrays, the engine's stages and the pipeline's buffers are each carved from
 * one allocation, so the total is exact up to the driver's own context memory.
 * out[] needs FC_MEM_FIELDS entries (bytes unless noted). */
enum {
  FC_MEM_FAST_ROWS = 0,        /* cached rows (+ optimizer state) [C, D+S] */
  FC_MEM_ID_SPACE = 1,         /* id/rank-space arrays: rank_of, rank_to_slot, aux, pending marks */
  FC_MEM_BITMAPS = 2,          /* residency / per-batch / free-slot bitmaps */
  FC_MEM_SLOT_SPACE = 3,       /* slot tables, per-slot lists, counters, pipeline index lists */
  FC_MEM_STAGING = 4,          /* write-back and admission stages in HBM */
  FC_MEM_SCRATCH = 5,          /* backward / scatter_update scratch (grown on demand) */
  FC_MEM_ALLOC_SLACK = 6,      /* rounding of the allocations to the 2 MiB device pages */
  FC_MEM_TOTAL_DEVICE = 7,     /* device memory the cache's allocations reserve: sum of the above */
  FC_MEM_PINNED_STAGING = 8,   /* pinned host staging of the write-back (not the slow tier) */
  FC_MEM_WB_STAGE_ROWS = 9,    /* rows per write-back stage buffer (count) */
  FC_MEM_ADMIT_STAGE_ROWS = 10,/* rows per admission stage buffer (count) */
  FC_MEM_FIELDS = 11
};
int fc_memory_bytes(fc_cache* h, int64_t* out, int32_t n_out);

/* Event-log payload of the last prepare (CacheEvent, cache_manager.py:78-99):
 * evicted ranks (descending) and admitted ranks (ascending), device -> host. */
int fc_last_events(fc_cache* h, int64_t* evicted_host, int64_t* admitted_host, void* stream);

/* flush (cache_manager.py:403-415): every dirty slot written back; rows stay. */
int fc_flush(fc_cache* h, void* stream, int64_t* rows_written);

/* mark_dirty (cache_manager.py:393-400). */
int fc_mark_dirty(fc_cache* h, const int64_t* slots_dev, int64_t n, void* stream);

/* select_evictions (cache_manager.py:205-216): slots of the `needed` largest
 * occupied ranks outside `protected`, in descending-rank order. */
int fc_select_evictions(fc_cache* h, int64_t needed, const int64_t* protected_dev, int64_t n_protected,
                        int64_t* slots_host, void* stream);

/* ---- frequency reorder ------------------------------------------------------ */
/* scan_frequencies + build_reorder (freq_stats.py:97-111, 136-148) on device:
 * counts = bincount(trace, minlength=num_ids) (int64), id_of = argsort(-counts,
 * stable) i.e. descending count, ties and unseen ids by ascending id, and
 * rank_of = its inverse (both int32). ids_dev: n ids, int64 if ids_bytes==8 else
 * int32. FC_ERR_ID_OUT_OF_RANGE names the smallest negative id, else the largest
 * id >= num_ids (freq_stats.py:82-90), in *bad_id. Synchronises `stream`. */
int fc_build_reorder(const void* ids_dev, int32_t ids_bytes, int64_t n, int64_t num_ids, int64_t* counts_dev,
                     int32_t* id_of_dev, int32_t* rank_of_dev, int64_t* bad_id, void* stream);

/* ---- lookups and updates ---------------------------------------------------- */
/* Pooled EmbeddingBag forward over cached rows (north star; semantics of
 * torch.nn.functional.embedding_bag; mean+psw = sum(w*row)/L, empty bag -> 0).
 * occurrence j uses row fast[unique_slots[inverse[j]]]. offsets == NULL means
 * one occurrence per bag (gather, cache_manager.py:418-420).
 * out: [n_bags, dim] fp32. offsets are int64 if offsets_bytes==8 else int32. */
int fc_pooled_forward(fc_cache* h, const int32_t* unique_slots, const int32_t* inverse, int64_t n,
                      const void* offsets, int32_t offsets_bytes, int64_t n_bags,
                      int32_t include_last_offset, const float* per_sample_weights, int32_t mode,
                      float* out, void* stream);

/* Rows of the unique ids (CacheStack.gather_unique, cache_manager.py:509-510). */
int fc_gather_rows(fc_cache* h, const int32_t* slots, int64_t n, float* out, void* stream);

/* apply_unique_update (cache_manager.py:517-523): fast[slot[p]] += add[p]; dirty. */
int fc_apply_unique_update(fc_cache* h, const int32_t* unique_slots, int64_t u, const float* add,
                           void* stream);

/* The simulator's deterministic update fused on device (simulator.py:246-260,433):
 * add[p][c] = ((hash24(id_p, salt)*2^-24 - 0.5) * count_p) * colw[c]. */
int fc_apply_synthetic_update(fc_cache* h, const int32_t* unique_ids, const int32_t* unique_counts,
                              const int32_t* unique_slots, int64_t u, uint64_t salt,
                              const float* colw, void* stream);

/* scatter_update (cache_manager.py:423-438): per-occurrence deltas accumulated in
 * batch order (bit-exact with np.add.at), every unique slot dirtied. */
int fc_scatter_update(fc_cache* h, const int32_t* unique_slots, const int32_t* inverse,
                      const int32_t* unique_counts, int64_t u, int64_t n, const float* deltas,
                      void* stream);

/* Fused backward of the pooled forward + sparse optimizer row update (north star
 * item 6): sort occurrences by unique row, segmented reduction of
 * grad_out[bag(j)] * coef_j, then SGD (w -= lr*g) or Adagrad
 * (G += g^2; w -= lr*g/(sqrt(G)+eps)) on the cached rows; rows dirtied. */
int fc_backward_update(fc_cache* h, const int32_t* unique_slots, const int32_t* inverse,
                       const int32_t* unique_counts, int64_t u, int64_t n,
                       const void* offsets, int32_t offsets_bytes, int64_t n_bags,
                       int32_t include_last_offset, const float* per_sample_weights, int32_t mode,
                       const float* grad_out, int32_t optim, float lr, float eps, void* stream);

/* ---- row-sharded exchange (multi-GPU, no reference counterpart: the reference's
 * sharding is column-wise only, sharding.py:62-118; this is the partitioned
 * scaling variant of SURVEY 8e/8f rank 2) ------------------------------------- */
typedef struct fc_router fc_router;  /* bitmap + scratch over a [world x S] routing key space */

int fc_router_create(int64_t num_ids, int32_t world, int32_t device, fc_router** out);
/* Table-wise placement (north star: tables sharded table-wise or column-wise): table t is the
 * id range [table_starts[t], table_starts[t+1]) (table_starts[0] = 0, [num_tables] = num_ids)
 * and belongs whole to rank table_owner[t]; an owner's local rows are its tables in table
 * order. fc_route then groups ids by owner and returns owner-local ids, as for row-wise.
 * Replaces the reference's table-wise placement, which it only plans and measures
 * (plan_tables_greedy / tablewise_imbalance, sharding.py:158-193): here the owners come
 * from that same greedy and the ids are actually routed to them. */
int fc_router_create_tables(int64_t num_ids, int32_t world, int32_t num_tables, const int64_t* table_starts_host,
                            const int32_t* table_owner_host, int32_t device, fc_router** out);
int fc_router_destroy(fc_router* r);

/* A requester's batch routed to row owners (owner = id % world, owner-local row =
 * id / world): unique ids grouped by owner, ascending within each owner, written as
 * owner-local ids to local_ids_dev (capacity n); inverse_dev[j] = position of ids[j]
 * in that list; owner_counts_host[o] = how many go to owner o; *unique = list length.
 * Synchronises `stream` (the counts size the all-to-all). */
int fc_route(fc_router* r, const void* ids_dev, int32_t ids_bytes, int64_t n, int32_t* local_ids_dev,
             int32_t* inverse_dev, int64_t* owner_counts_host, int64_t* unique, void* stream);

/* Pooled EmbeddingBag forward over a dense row buffer: occurrence j uses
 * rows[inverse[j]] (the rows the owners sent back, in routing order). */
int fc_pool_rows(const float* rows_dev, int32_t dim, const int32_t* inverse_dev, int64_t n, const void* offsets,
                 int32_t offsets_bytes, int64_t n_bags, int32_t include_last_offset,
                 const float* per_sample_weights, int32_t mode, float* out, void* stream);

/* The backward of fc_pool_rows: one gradient row per routed unique id,
 * grad_unique[p] = sum over occurrences j with inverse[j] == p of coef_j * grad_out[bag(j)]
 * (deterministic order), ready to be sent to the owners. */
int fc_route_grads(fc_router* r, const int32_t* inverse_dev, int64_t u, int64_t n, const void* offsets,
                   int32_t offsets_bytes, int64_t n_bags, int32_t include_last_offset,
                   const float* per_sample_weights, int32_t mode, const float* grad_out, int32_t dim,
                   float* grad_unique, void* stream);

/* Owner side of the row-sharded forward fused with the return exchange: the cached row
 * of received id i (requester r = the segment of i in seg_dev[0..world]) is written
 * straight into requester r's receive buffer dst_ptrs_dev[r] (a peer pointer over NVLink,
 * from fc_ipc_open, or local memory for r == self) at row dst_off_dev[r] + (i - seg[r]).
 * Order it before a stream-ordered barrier (a tiny all-reduce) before requesters read. */
int fc_pool_to_peers(fc_cache* h, const int32_t* unique_slots, const int32_t* inverse, int64_t n,
                     const int64_t* seg_dev, int32_t world, float* const* dst_ptrs_dev, const int64_t* dst_off_dev,
                     void* stream);
/* The backward's mirror: an owner pulls the gradient row of each received id i
 * (requester r = the segment of i) from src_ptrs_dev[r] at row src_off_dev[r] + (i - seg[r])
 * over peer memory into out [n, dim]; order it after a barrier that follows the
 * requesters' writes. */
int fc_gather_from_peers(const float* const* src_ptrs_dev, const int64_t* src_off_dev, const int64_t* seg_dev,
                         int32_t world, int64_t n, int32_t dim, float* out, void* stream);
/* Column-wise split (the reference's sharding.py:62-118), forward fused with its all-to-all
 * (the exchange sharding.py:133-146 only accounts for): this rank's pooled column slice of
 * global occurrence i (bag size 1; requester r = the segment of i in seg_dev[0..world]) is
 * written straight into requester r's output dst_ptrs_dev[r] (peer pointer over NVLink) at
 * row dst_off_dev[r] + (i - seg[r]), columns [col, col + dim) of rows ld floats wide; psw
 * (optional, per global occurrence) scales the row. dim, ld and col multiples of 4. */
int fc_pool_cols_to_peers(fc_cache* h, const int32_t* unique_slots, const int32_t* inverse, int64_t n,
                          const int64_t* seg_dev, int32_t world, float* const* dst_ptrs_dev,
                          const int64_t* dst_off_dev, int64_t ld, int64_t col, const float* per_sample_weights,
                          void* stream);
/* Its backward mirror: columns [col, col + dim) of every requester's gradient rows
 * (src_ptrs_dev[r], rows ld floats wide, from row src_off_dev[r]) gathered over peer memory
 * into out [n, dim] in global occurrence order, ready for fc_backward_update. */
int fc_gather_cols_from_peers(const float* const* src_ptrs_dev, const int64_t* src_off_dev, const int64_t* seg_dev,
                              int32_t world, int64_t n, int32_t dim, int64_t ld, int64_t col, float* out,
                              void* stream);
/* CUDA IPC plumbing for the peer pointers. handle_out: FC_IPC_HANDLE_BYTES opaque bytes
 * (the allocation's cudaIpcMemHandle_t + the pointer's offset inside it, so pointers into a
 * caching allocator's segment export correctly); fc_ipc_open returns the same address in
 * the importing process; fc_ipc_close takes the pointer fc_ipc_open returned. */
#define FC_IPC_HANDLE_BYTES 128
int fc_ipc_handle(void* dev_ptr, void* handle_out);
int fc_ipc_open(const void* handle, int32_t device, void** dev_ptr_out);
int fc_ipc_close(void* dev_ptr);

#ifdef __cplusplus
}
#endif
#endif /* FREQCACHE_B200_H */
