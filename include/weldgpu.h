/* weldgpu.h -- C ABI of libweldgpu.so, the B200 executor under the Weld IR's
 * data-parallel core (`for(vector, builders, func)` + the five builders).
 *
 * The reference (weldmill, pure Python) has no native boundary: its executor
 * seam is the module function
 *     weldmill.engine.evaluate(e, env, config, externs) -> (Value, EvalStats)
 *     /root/reference/pkg/src/weldmill/engine/run.py:1008-1074
 * imported by name at api.py:23 and called at api.py:374.  The Python package
 * paper_1709_06416_b200 keeps that exact signature and binds this library
 * with ctypes.  Each entry point below says which
 * reference code path it replaces.
 *
 * Conventions: every function returns 0 on success, -1 on failure with the
 * message available from wg_last_error() (thread-local).  Device addresses
 * are plain uint64_t; no exceptions cross the ABI; no torch types.
 */
#ifndef WELDGPU_H
#define WELDGPU_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- process / device ------------------------------------------------- */
const char* wg_last_error(void);
int wg_version(void);
int wg_device_count(int* n);
/* Replaces the per-evaluate worker pool set-up (_Pool, run.py:261-284): one
 * device and one non-blocking stream per process. */
int wg_init(int device);
int wg_sm_count(int* n);
int wg_stream(uint64_t* stream);
int wg_sync(void);

/* ---- columnar buffer manager (replaces Python lists + _Runtime.alloc,
 *      run.py:184-228, builders.py:59-106) --------------------------------- */
int wg_alloc(uint64_t bytes, uint64_t* dptr);
int wg_free(uint64_t dptr);
int wg_mem_trim(void);
int wg_mem_stats(uint64_t* live, uint64_t* peak);
int wg_mem_reset_peak(void);
int wg_memset(uint64_t dptr, int value, uint64_t bytes);
int wg_h2d(uint64_t dst, const void* src, uint64_t bytes);
int wg_d2h(void* dst, uint64_t src, uint64_t bytes);
int wg_d2h_async(void* dst, uint64_t src, uint64_t bytes);
int wg_d2d(uint64_t dst, uint64_t src, uint64_t bytes);
int wg_host_alloc(uint64_t bytes, void** p);
int wg_host_free(void* p);
int wg_host_register(void* p, uint64_t bytes);
int wg_host_unregister(void* p);

/* ---- runtime errors (replaces the EvalError raises inside the loop body,
 *      run.py:411-425, 693-710; builders.py:413-417) ------------------------ */
int wg_error_ptr(uint64_t* p);
int wg_read_error(int64_t* code, int64_t* info);
/* the error word captured by the last wg_dict_finish_small (same sync as its count), then cleared */
int wg_last_sync_error(int64_t* code, int64_t* info);
/* device -> host copy plus the error-word check, one stream synchronisation */
int wg_d2h_checked(void* dst, uint64_t src, uint64_t bytes, int64_t* code, int64_t* info);

/* ---- loop compilation and launch (replaces _compile_inner/_compile_for,
 *      run.py:560-983: the closure network becomes one NVRTC-compiled
 *      sm_100a kernel per fused outer `for`) -------------------------------- */
int wg_compile(const char* src, const char* name, int nheaders, const char* const* header_srcs,
               const char* const* header_names, int nopts, const char* const* opts, uint64_t* module_out,
               char* log_buf, uint64_t log_cap);
int wg_compile_check(const char* src, const char* name, int nheaders, const char* const* header_srcs,
                     const char* const* header_names, int nopts, const char* const* opts, uint64_t* cubin_bytes,
                     char* log_buf, uint64_t log_cap);
int wg_compile_ptx(const char* src, const char* name, int nheaders, const char* const* header_srcs,
                   const char* const* header_names, int nopts, const char* const* opts, char* ptx_out,
                   uint64_t ptx_cap, uint64_t* ptx_size, char* log_buf, uint64_t log_cap);
int wg_module_load(const char* image, uint64_t* module_out);
int wg_module_function(uint64_t module, const char* name, uint64_t* fn);
int wg_occupancy(uint64_t fn, int block, int dyn_smem, int* blocks_per_sm);
int wg_launch(uint64_t fn, uint32_t grid, uint32_t block, uint32_t dyn_smem, const void* params,
              uint64_t params_size);

/* ---- builder result() helpers ------------------------------------------
 * dictmerger table init/compaction: DictMergerState.result, builders.py:380-392
 * order_key transform + stable sort: order_key builders.py:496-507, ToVec
 *   run.py:737-747, Sort run.py:723-735
 * run starts: GroupBuilderState.result, builders.py:478-493 */
int wg_table_init(uint64_t table, uint64_t nslots, int slot_words, const uint64_t* pattern);
int wg_table_compact(uint64_t table, uint64_t nslots, int slot_words, int mode, const uint64_t* out_words, int nout,
                     uint64_t* count_out);
/* Small dictmerger result in one launch: occupied slots -> entries sorted by
 * the order_key tuple -> typed key/value columns (DictMergerState.result,
 * builders.py:380-392 + order_key :496-507).  key_desc = 4 ints per key leaf
 * (word, shift, width, kind); counters = the table's {distinct, spilled}
 * words (device).  *count_out > 4096 means nothing was written; ~0 means
 * spilled merges must be replayed first. */
int wg_dict_finish_small(uint64_t table, uint64_t nslots, int slot_words, int mode, int nw, int nkl,
                         const int* key_desc, int nvl, const int* val_kinds, const uint64_t* outs,
                         uint64_t counters, uint64_t* count_out);
int wg_order_key(uint64_t src, int kind, uint64_t n, uint64_t perm, uint64_t dst);
int wg_iota_u32(uint64_t dst, uint64_t n);
/* offsets[j] = j * step of vec[vec[T]] results built from fixed-length vectors
 * (VecBuilderState.result, builders.py:274-283, for nested element types) */
int wg_iota_i64(uint64_t dst, uint64_t n, int64_t step);
/* exclusive scan of n i64 per-tile append counts -> tile offsets; *total (device) = sum
 * (two-pass order-preserving appends: VecBuilderState.result order, builders.py:274-283) */
int wg_exclusive_scan_i64(uint64_t src, uint64_t dst, uint64_t n, uint64_t total);
/* reallocation accounting of an unhinted vecbuilder's scan-mode launch
 * (VecBuilderState.merge, builders.py:256-272): coff[c] = output position of
 * chunk c's first append (nch grain-wide chunks), *total = the launch's
 * appends (device).  out (device u64[4]): sum of doublings and of final
 * capacities over interior chunks 1..nch-2, then the first and last chunk's
 * append counts. */
int wg_seg_stats(uint64_t coff, uint64_t nch, uint64_t total, uint64_t out);
/* the +0.0 key of a sorted float dictionary key column (width 4 or 8) becomes
 * -0.0 when a -0.0 key was merged first (DictMergerState._upsert keeps the
 * first-inserted key object, builders.py:346-351) */
int wg_neg_zero(uint64_t col, uint64_t n, int width);
int wg_sort_pairs(uint64_t keys_in, uint64_t vals_in, uint64_t keys_out, uint64_t vals_out, uint64_t n, int begin_bit,
                  int end_bit);
int wg_gather(uint64_t src, uint64_t perm, uint64_t dst, uint64_t n, int width);
int wg_narrow(uint64_t src, uint64_t dst, int width, uint64_t n);
int wg_widen(uint64_t src, uint64_t dst, int width, uint64_t n);
int wg_run_starts(const uint64_t* key_words, int kw, uint64_t n, uint64_t starts_out, uint64_t* nruns);
int wg_group_finish1(uint64_t keys, int key_kind, uint64_t vals, int val_width, uint64_t n, uint64_t ukeys_out,
                     uint64_t offs_out, uint64_t vals_out, uint64_t* K_out);

/* ---- synthetic inputs and measurement (bench.py; no reference analogue) -- */
int wg_gen_column(uint64_t dst, uint64_t n, uint64_t row0, int dist, int width, uint64_t seed, uint64_t col,
                  int64_t lo, uint64_t span, double flo, double fhi, double div, int ncat, const double* cum,
                  const int64_t* vals);
int wg_mul_inplace_f64(uint64_t a, uint64_t b, uint64_t n);
int wg_flush_l2(uint64_t buf, uint64_t bytes, uint32_t salt);
int wg_event_create(uint64_t* ev);
int wg_event_record(uint64_t ev);
int wg_event_elapsed_ms(uint64_t start, uint64_t stop, float* ms);
int wg_event_destroy(uint64_t ev);
/* Per-launch device timing: while enabled, every kernel the library launches
 * (fixed-function and NVRTC loop kernels) is bracketed by CUDA events on its
 * stream and recorded under its name; enabling clears the records. */
int wg_prof_enable(int on);
int wg_prof_count(int* n);
int wg_prof_record(int i, char* name, int cap, float* ms);
/* Copy/compute overlap for host-resident inputs (executor streaming path). */
int wg_stream_select(int which);
int wg_stream_wait_event(uint64_t ev);
int wg_sync_all(void);

/* ---- multi-GPU combine (row-partitioned evaluation) -------
 * The reference folds per-chunk builder partials at result() --
 * merger builders.py:314-328, dictmerger :380-392, vecmerger :435-450,
 * groupbuilder :478-493 -- on one host.  Across GPUs each rank's partial is
 * exchanged with these entry points (NCCL over NVLink, libnccl.so.2 loaded
 * at wg_nccl_init) and folded by device kernels.
 *
 * wg_partition: stable split of n rows into nsplit+1 destinations by the
 *   order key (builders.py:496-507) of the first key leaf against ascending
 *   splitter order keys; every column is scattered so each destination's rows
 *   are contiguous and in input order; counts_out (host) gets the
 *   per-destination row counts. */
int wg_partition(uint64_t key_col, int key_kind, const uint64_t* splitters, int nsplit, int ncols,
                 const uint64_t* cols_in, const uint64_t* cols_out, const int* widths, uint64_t n,
                 uint64_t* counts_out);
int wg_nccl_unique_id(char* out, int cap);
int wg_nccl_init(int rank, int world, const char* id_bytes);
int wg_nccl_finalize(void);
int wg_nccl_allgather(uint64_t send, uint64_t recv, uint64_t bytes);
int wg_nccl_allreduce(uint64_t send, uint64_t recv, uint64_t count, int kind, int op);
int wg_nccl_sendrecv(int nsend, const uint64_t* send_ptr, const uint64_t* send_bytes, const int* send_peer,
                     int nrecv, const uint64_t* recv_ptr, const uint64_t* recv_bytes, const int* recv_peer);

#ifdef __cplusplus
}
#endif
#endif /* WELDGPU_H */
