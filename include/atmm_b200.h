/*
 * atmm_b200.h -- C ABI of the B200-native ATMM operator (libatmm_b200.so).
 *
 * Drop-in boundary for the reference's ATMM hot path (loraserve, header-only
 * C++ under /root/reference/proj/include/loraserve).  The reference has no C
 * ABI; each entry point below names the reference function it replaces
 * (file:line, paths relative to proj/include/loraserve/).  The header-only
 * C++ shim include/loraserve_b200.hpp restores the reference's C++
 * signatures and exception types on top of this ABI.
 *
 * Conventions
 *  - Every function returns an int status (ATMM_OK == 0, else an ATMM_ERR_*
 *    code that maps 1:1 onto the reference's exception classes,
 *    errors.hpp:10-61); the message is in atmm_last_error() (thread-local).
 *  - No function throws; all are safe to call from C.
 *  - Device-pointer entry points are stream-ordered on the caller's
 *    cudaStream_t (passed as void*; NULL = legacy default stream) and never
 *    synchronize.  *_host entry points take host buffers and are synchronous.
 *  - Matrices are row-major, `ld` in elements.  Row-vector convention of the
 *    reference: y = x . W, down is d_in x r, up is r x d_out (adapter.hpp:15-16).
 *  - Compute: bf16 operands, fp32 accumulation on tcgen05 tensor cores.
 *    There is no CPU fallback: without an sm_100 device the compute calls
 *    return ATMM_ERR_NO_DEVICE.
 */
#ifndef ATMM_B200_H_
#define ATMM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ATMM_ABI_VERSION 2

/* Status codes <-> loraserve exception classes (errors.hpp). */
enum {
  ATMM_OK = 0,
  ATMM_ERR_SHAPE = 1,           /* ShapeError            errors.hpp:16-25 */
  ATMM_ERR_CONFIG = 2,          /* ConfigError           errors.hpp:27-30 */
  ATMM_ERR_MODE = 3,            /* ModeError             errors.hpp:32-36 */
  ATMM_ERR_IO = 4,              /* IoError               errors.hpp:38-41 */
  ATMM_ERR_PARSE = 5,           /* ParseError            errors.hpp:43-52 */
  ATMM_ERR_UNKNOWN_ADAPTER = 6, /* UnknownAdapterError   errors.hpp:54-62 */
  ATMM_ERR_CUDA = 7,            /* CUDA runtime / launch failure          */
  ATMM_ERR_NO_DEVICE = 8,       /* no sm_100 device: there is no fallback */
  ATMM_ERR_INTERNAL = 9
};

/* Element types for activations / outputs / weights. */
enum { ATMM_BF16 = 0, ATMM_F32 = 1 };

const char* atmm_last_error(void);
int atmm_abi_version(void);
/* Number of sm_100 devices visible (0 on a CPU-only host; never fails). */
int atmm_device_count(void);

/* Algorithmic FLOP accounting (flops.hpp:10-24): a thread-local counter of
 * the FLOPs (2 per multiply-add) the reference's GEMMs would count for the
 * same calls -- padding-free, heterogeneous ranks at their own rank.  Every
 * compute entry point below adds to it on success (atmm_bypass_apply: the
 * plan's sum_seg 2 ns r (d_in + d_out); merge: 2 d_in d_out r per layer; GEMM:
 * 2 m n k; forward: per layer 2 n d^2 + the bypass). */
uint64_t atmm_flops_read(void);
void atmm_flops_reset(void);
/* Host-only: the bypass FLOPs of one batch, sum over plan_batch segments of
 * 2 ns r_a (d_in + d_out) (test_batch.cpp:96-128).  UnknownAdapter if a
 * segment's id is not in adapter_ids. */
int atmm_bypass_flops(const int32_t* assignment, int64_t n, const int32_t* adapter_ids, const int64_t* adapter_ranks,
                      int64_t num_adapters, int64_t d_in, int64_t d_out, uint64_t* flops);

/* ===================================================================== */
/* Planner                                                                */
/* ===================================================================== */

/* plan_batch (batch.hpp:28-42): stable group-by of rows per adapter id,
 * segments in ascending id order.  Output is CSR: seg_adapter[S],
 * seg_offsets[S+1], row_index[n] (caller-allocated, capacity n / n+1 / n).
 * Empty assignment -> ATMM_ERR_CONFIG. */
int atmm_plan_batch(const int32_t* assignment, int64_t n, int32_t* seg_adapter,
                    int64_t* seg_offsets, int64_t* row_index, int64_t* num_segments);

/* ===================================================================== */
/* Tiling configuration and the shape-keyed table (tiling.hpp)            */
/* ===================================================================== */

/* cfg = {outer_m, outer_n, outer_k, inner_m, inner_n, inner_k}
 * (TilingConfig, tiling.hpp:22-65).  On B200 the edges are read as:
 *   outer_m  rows per cluster tile (segment rows are cut into tiles of this)
 *   outer_k  K slice per CTA  -> cluster size C = ceil(d_in / outer_k)
 *   outer_n  expand N chunk per tcgen05.mma (<= 256 columns)
 *   inner_*  tcgen05 instruction shape (M=128 / N granule / K stage = 64),
 *            validated like the reference but otherwise informational. */
int atmm_config_valid(const int32_t cfg[6]); /* structurally_valid tiling.hpp:40-48 -> 1/0 */
int atmm_m_bucket_of(int64_t m);             /* m_bucket_of tiling.hpp:76-79 */

typedef struct atmm_table atmm_table;
/* TilingTable() / TilingTable(default) (tiling.hpp:160-162).  NULL default =
 * the reference default {64,32,32,32,32,32}; a default-constructed table
 * resolves its default through the B200 heuristic. */
int atmm_table_create(const int32_t* default_cfg, atmm_table** out);
void atmm_table_destroy(atmm_table* t);
/* TilingTable::insert (tiling.hpp:164-167).  sm100 (nullable) = explicit
 * B200 launch parameters {tile_m, cluster, bn, stages, path} stored beside
 * the reference entry (the JSON "sm100" object):
 *   tile_m  rows per tile (1..128)      cluster  CTAs per tile (1..16)
 *   bn      expand N chunk (64..256)    stages   shrink ring depth (0 = auto)
 *   path    ATMM_PATH_* kernel choice (ATMM_PATH_AUTO picks by tile rows;
 *           ATMM_PATH_STREAM runs the whole plan as ONE persistent launch). */
enum { ATMM_PATH_AUTO = 0, ATMM_PATH_A2A = 1, ATMM_PATH_SPLIT = 2, ATMM_PATH_FUSED = 3, ATMM_PATH_STREAM = 4 };
int atmm_table_insert(atmm_table* t, int32_t m_bucket, int32_t k, int32_t n,
                      const int32_t cfg[6], int64_t measured_ns, const int32_t* sm100);
/* TilingTable::set_default (tiling.hpp:169); sm100 (nullable) = the default's
 * B200 launch (JSON "default_sm100"), used for shapes the table misses;
 * sm100 = {0, ...} makes misses resolve through the built-in B200 heuristic
 * (JSON "default_sm100": "heuristic"). */
int atmm_table_set_default(atmm_table* t, const int32_t cfg[6], const int32_t* sm100);
/* TilingTable::lookup (tiling.hpp:181-199): exact -> nearest same-(k,n)
 * bucket within 32 (ties to the smaller bucket) -> default. */
int atmm_table_lookup(const atmm_table* t, int64_t m, int64_t k, int64_t n, int32_t cfg_out[6]);
int atmm_table_size(const atmm_table* t, int64_t* size);
/* The entry lookup(m, k, n) hits (exact or nearest bucket within 32):
 * *found = 1 and its B200 launch, else *found = 0 (the default applies). */
int atmm_table_find(const atmm_table* t, int64_t m, int64_t k, int64_t n, int32_t launch_out[5], int* found);
/* The B200 launch parameters the table resolves for the fused bypass of a
 * segment of m rows at (d_in, rank, d_out): {tile_m, cluster, bn, stages,
 * path}.  t == NULL gives the built-in heuristic. */
int atmm_table_resolve_launch(const atmm_table* t, int64_t m, int64_t d_in, int64_t rank,
                              int64_t d_out, int32_t launch_out[5]);
/* TilingTable::save / load (tiling.hpp:201-249): same JSON schema,
 * {"default":[6], "entries":[{m_bucket,k,n,config[6],ns[,sm100]}]}. */
int atmm_table_save(const atmm_table* t, const char* path);
int atmm_table_load(const char* path, atmm_table** out);
/* candidate_configs / default_candidates (tiling.hpp:88-149): writes up to
 * cap configs (6 ints each) and the total count. */
int atmm_candidate_configs(size_t cache_budget_bytes, size_t scalar_width, int32_t* out,
                           size_t cap, size_t* count);
int atmm_default_candidates(size_t cache_budget_bytes, size_t scalar_width, int32_t* out,
                            size_t cap, size_t* count);

/* ===================================================================== */
/* Fixture matrices (matrix.hpp:183-218): little-endian u32 rows, u32 cols, */
/* u8 scalar width (4), row-major fp32 payload -- the reference's format.   */
/* ===================================================================== */
int atmm_matrix_save(const char* path, int64_t rows, int64_t cols, const float* data);
/* out may be NULL (dims only); else capacity >= rows * cols floats. */
int atmm_matrix_load(const char* path, int64_t* rows, int64_t* cols, float* out, int64_t capacity);
/* A fixture directory's manifest.json (model_io.hpp:25-69 layout): layer
 * count, hidden dim and the adapters' ids / ranks (first `capacity`). */
int atmm_fixture_info(const char* dir, int64_t* num_layers, int64_t* hidden_dim, int64_t* num_adapters,
                      int32_t* ids, int64_t* ranks, int64_t capacity);

/* ===================================================================== */
/* Adapter registry (adapter.hpp:18-110, device resident)                 */
/* ===================================================================== */

typedef struct atmm_registry atmm_registry;
/* A registry holds the LoRA factors of every adapter for `num_layers`
 * layers of one d_in x d_out projection, in HBM, in the tcgen05 operand
 * layouts.  device = CUDA ordinal. */
int atmm_registry_create(int device, int64_t num_layers, int64_t d_in, int64_t d_out,
                         atmm_registry** out);
void atmm_registry_destroy(atmm_registry* r);
/* LoraAdapter(...) (adapter.hpp:26-51) + AdapterSet::emplace: host fp32
 * factors down [L][d_in x r] and up [L][r x d_out]; scale s multiplies the
 * adapter's contribution (the reference's implicit s = 1).  Any rank
 * 1 <= r < hidden (adapter.hpp:30-31; r <= 128 is also accepted on smaller
 * layers): r <= 128 is one slot; a larger rank is stored as 128-rank chunk
 * slots that every bypass applies as extra passes over the same Y rows
 * (separate launches, one bf16 rounding of Y per pass) and merge / delta_w
 * sum chunk by chunk.  Rank-chunked adapters are not taken by put_async,
 * put_combined, precise registries or the fused layer forward (ConfigError).
 * Re-putting an id replaces it. */
int atmm_registry_put(atmm_registry* r, int32_t adapter_id, int64_t rank, const float* down,
                      const float* up, float scale);
/* Asynchronous adapter swap (serving.hpp:38-74 mode_switch, the paper's
 * adapter swap): same factors and result as atmm_registry_put, but the H2D
 * copy (pinned host memory for a truly async copy), the fp32 -> bf16
 * operand-layout packing (a device kernel) and the release of a replaced
 * slot's memory are all ordered on `stream`; work launched later on that
 * stream sees the new factors. */
int atmm_registry_put_async(atmm_registry* r, int32_t adapter_id, int64_t rank, const float* down,
                            const float* up, float scale, void* stream);
/* load_model_fixture (model_io.hpp:71-114), adapter part: reads the
 * fixture's manifest.json and binary matrix files (matrix.hpp:183-218) and
 * puts every adapter (all layers) into the registry; the registry must match
 * the fixture (num_layers, d_in == d_out == hidden_dim).  IoError on a bad or
 * truncated file, ShapeError on mismatched factors. */
int atmm_registry_load_fixture(atmm_registry* r, const char* dir, int64_t* num_adapters);
int atmm_registry_remove(atmm_registry* r, int32_t adapter_id);
/* Mixture / deLoRA branch (model.hpp:252-328): a slot whose
 * factors are the rank-concatenation of existing adapters,
 *   down = [down_1 | down_2 | ...],  up = [s_1 sign_1 up_1 ; s_2 sign_2 up_2 ; ...],
 * so ONE fused bypass adds sum_i sign_i s_i (x.down_i).up_i with a single
 * rounding into Y (e.g. parts {a, merged} signs {+1, -1}: own adapter minus
 * the cancel branch of the merged adapter).  Sum of padded ranks <= 128
 * (ConfigError otherwise: the Python MixturePlan then runs those guests in
 * the two-pass form, own branch then cancel branch).
 * Signs / scales of +-1 (and powers of two) are folded exactly. */
int atmm_registry_put_combined(atmm_registry* r, int32_t new_id, int64_t n_parts, const int32_t* part_ids,
                               const float* part_signs);
/* adapter_at (adapter.hpp:106-110): 1 if present, 0 if not. */
int atmm_registry_contains(const atmm_registry* r, int32_t adapter_id);
int atmm_registry_rank(const atmm_registry* r, int32_t adapter_id, int64_t* rank);
/* Bytes of adapter factors resident in HBM (bf16 operand layouts). */
int atmm_registry_bytes(const atmm_registry* r, int64_t* bytes);

/* ===================================================================== */
/* Fused batched-LoRA bypass (batch.hpp:48-81 + model.hpp:239-241)        */
/* ===================================================================== */

typedef struct atmm_plan atmm_plan;
/* plan_batch + tile/launch grouping for one batch on one registry.
 * Unknown ids -> ATMM_ERR_UNKNOWN_ADAPTER (fail fast like
 * forward_unmerged, model.hpp:226-228).  table may be NULL (heuristic). */
int atmm_plan_create(atmm_registry* r, const int32_t* assignment, int64_t n,
                     const atmm_table* table, atmm_plan** out);
/* plan_batch over a subset of the rows: routed entry i (adapter
 * assignment[i]) is row rows[i] of X / Y, which have n_rows rows (rows
 * distinct).  Used for mixture mode, where only the guest rows (those not
 * served by the merged weights, model.hpp:273-280) take a bypass. */
int atmm_plan_create_mapped(atmm_registry* r, const int32_t* assignment, const int32_t* rows, int64_t n,
                            int64_t n_rows, const atmm_table* table, atmm_plan** out);
/* A plan whose every segment runs `launch` {tile_m, cluster, bn, stages,
 * path} instead of the table's (the tuner's candidates; path-coverage tests). */
int atmm_plan_create_launch(atmm_registry* r, const int32_t* assignment, int64_t n, const int32_t launch[5],
                            atmm_plan** out);
void atmm_plan_destroy(atmm_plan* p);
/* Plan flags (no reference counterpart: a launch-ordering promise).
 * ATMM_PLAN_X_READY: the X handed to every apply of this plan is complete
 * before the launch preceding the apply on its stream starts (e.g. the
 * bypass follows the base GEMM Y = X.W, which reads X and writes Y).  The
 * fused kernels then gather X before griddepcontrol.wait, under the tail of
 * that launch; Y is still read only after it completes.  Results are
 * unchanged; breaking the promise races on X. */
#define ATMM_PLAN_X_READY 1u
/* ATMM_PLAN_NO_OVERLAP: never start an apply's X / Y loads under the
 * preceding launch.  By default the launcher does so for the all-to-all
 * kernel when it can prove safety: that kernel releases its successor only
 * after its own predecessor completed, so at most the immediately preceding
 * launch on the stream can still run, and the apply proceeds early only when
 * that launch is an all-to-all bypass whose X / Y bytes are disjoint from
 * this apply's (consecutive independent batches overlap; Y_i -> X_i+1 chains
 * keep the full dependency).  The split path's shrink likewise computes under
 * the preceding bypass launch when that launch's Y writes miss this apply's X
 * (it reads only X, the factors and a scratch set private to this apply; it
 * waits and releases the expand at its end).  Under stream capture the predecessor is also
 * matched by graph node.  Not visible to the check: a FOREIGN kernel launched
 * with the programmatic-stream-serialization attribute between two eager
 * applies on one stream -- set this flag when a caller does that. */
#define ATMM_PLAN_NO_OVERLAP 2u
int atmm_plan_set_flags(atmm_plan* p, uint32_t flags);
/* Process-wide counters: all-to-all bypass launches issued, and how many of
 * them started their X / Y loads early (ATMM_PLAN_NO_OVERLAP above). */
int atmm_overlap_stats(int64_t* a2a_launches, int64_t* early_launches);
/* The same for split-path applies: shrink + expand pairs issued, and how many
 * shrinks computed under the preceding launch. */
int atmm_split_overlap_stats(int64_t* split_launches, int64_t* early_launches);
/* Routing tables actually uploaded (for bit-exact routing checks):
 * seg_adapter[S], seg_offsets[S+1], row_index[n]. */
int atmm_plan_routing(const atmm_plan* p, int32_t* seg_adapter, int64_t* seg_offsets,
                      int64_t* row_index, int64_t* num_segments);
/* JSON description of the resolved launch groups (cluster, bn, stages,
 * ring depths, shared memory, TMEM columns) into buf (NUL-terminated). */
int atmm_plan_describe(const atmm_plan* p, char* buf, size_t cap);
/* Number of kernel launches / cluster tiles / CTAs the plan issues. */
int atmm_plan_stats(const atmm_plan* p, int64_t* launches, int64_t* tiles, int64_t* ctas);

/* Y[row, :] += scale * s_a * (X[row, :] . down_a[layer]) . up_a[layer]
 * for every row, a = assignment[row]: ONE pass, shrink+expand fused, the
 * rank-r intermediate kept on chip, the residual add fused in the epilogue.
 * X: n x d_in bf16, ldx >= d_in (rows that are not 16-byte aligned --
 * odd d_in, offset views -- are staged into a padded copy first, stream
 * ordered); Y: n x d_out, y_dtype ATMM_BF16 or ATMM_F32, any ldy >= d_out.  scale = -1 gives the deLoRA cancel branch
 * (model.hpp:315-321).  Device pointers, stream-ordered. */
int atmm_bypass_apply(const atmm_plan* p, int64_t layer, const void* x, int64_t ldx, void* y,
                      int64_t ldy, int y_dtype, float scale, void* stream);

/* `count` (1..8) independent applications of one plan -- call c computes
 * ys[c][row] += scale * s_a * (xs[c][row] . down_a[layers[c]]) . up_a[layers[c]]
 * -- as ONE launch when every launch group runs the all-to-all kernel (e.g.
 * the q / k / v projections of a decoder layer: same tokens and adapters,
 * per-projection factors stored as separate layers of the registry), else one
 * launch per call.  The calls must not write each other's inputs. */
int atmm_bypass_apply_group(const atmm_plan* p, int64_t count, const int64_t* layers, const void* const* xs,
                            int64_t ldx, void* const* ys, int64_t ldy, int y_dtype, float scale, void* stream);

/* run_bypass (batch.hpp:48) with host buffers: out = bypass(x), fp32 in and
 * out.  A precise registry computes it fp32-faithfully (atmm_bypass_apply_f32),
 * otherwise x is rounded to bf16 on the device.  Synchronous. */
int atmm_run_bypass_host(atmm_registry* r, const float* x, int64_t n,
                         const int32_t* assignment, int64_t layer, const atmm_table* table,
                         float* out);
/* The unmerged-forward residual site (model.hpp:239-241) end to end with
 * host buffers: H2D x and y, fused bypass into y, D2H y.  bf16 host
 * buffers (pinned if the caller wants full PCIe bandwidth).  Uses the
 * plan's device and the given stream; synchronizes on it. */
int atmm_bypass_residual_host_bf16(const atmm_plan* p, int64_t layer, const uint16_t* x_host,
                                   uint16_t* y_host, float scale, void* stream);

/* Serving form of the above: `count` micro-batches on the same plan, each with
 * its own host buffers (pinned for overlap), pipelined over two streams and
 * two device staging slots so the H2D of batch i+1 overlaps the kernel and
 * the D2H of batch i.  Returns when every y_hosts[i] holds its result. */
int atmm_bypass_residual_host_bf16_pipelined(const atmm_plan* p, const int64_t* layers,
                                             const uint16_t* const* x_hosts,
                                             uint16_t* const* y_hosts, int64_t count,
                                             float scale);
/* run_bypass (batch.hpp:48) end to end with bf16 HOST buffers, `count`
 * independent batches pipelined (H2D of one, compute of another, D2H of a
 * third): out_hosts[i] = bypass(x_hosts[i]) for layer layers[i] (a fresh
 * output, like run_bypass's returned matrix).  Pinned host memory for
 * overlap. */
int atmm_run_bypass_host_bf16_pipelined(const atmm_plan* p, const int64_t* layers, const uint16_t* const* x_hosts,
                                        uint16_t* const* out_hosts, int64_t count);

/* ===================================================================== */
/* Merge / unmerge  W +-= s . down . up   (model.hpp:120-188)             */
/* ===================================================================== */

/* W (d_in x d_out, w_dtype ATMM_F32 or ATMM_BF16, in place, address
 * stable) += sign * s_a * down_a[layer] . up_a[layer].  sign = +1 merges,
 * -1 unmerges.  Device pointer, stream-ordered. */
int atmm_merge_apply(atmm_registry* r, int32_t adapter_id, int64_t layer, void* w,
                     int64_t ldw, int w_dtype, float sign, void* stream);
/* delta_w (model.hpp:130-140) with a host output: out = s_a * down . up. */
/* merge / unmerge of ALL layers [layer0, layer0 + num_layers) in ONE launch
 * (model.hpp:144-188, the mode switch's one-shot merge): layer l's W is at
 * w + (l - layer0) * w_layer_stride elements.  One persistent grid streams
 * every layer's W through shared memory (TMA, 3-D tensor map). */
int atmm_merge_apply_layers(atmm_registry* r, int32_t adapter_id, int64_t layer0, int64_t num_layers, void* w,
                            int64_t ldw, int64_t w_layer_stride, int w_dtype, float sign, void* stream);
int atmm_delta_w_host(atmm_registry* r, int32_t adapter_id, int64_t layer, float* out);

/* ModelState (model.hpp:104-112) + merge / unmerge / mode_switch on device
 * weights.  A state binds the registry to the model's weights W (all
 * num_layers of the registry, layer l at w + l * w_layer_stride elements,
 * w_dtype ATMM_BF16 or ATMM_F32) and enforces the reference's mode contract:
 *   merge    (model.hpp:144-165) requires Unmerged, else ATMM_ERR_MODE;
 *   unmerge  (model.hpp:167-188) requires Merged/Mixture of that adapter;
 *   mode_switch (serving.hpp:38-74) issues the minimal sequence of one-shot
 *            (all-layer, one-launch) un/merges; Merged <-> Mixture of the same
 *            adapter touches no weights.  `launches` = weight rewrites issued.
 * Stream-ordered; W must stay allocated (address-stable) while bound. */
enum { ATMM_MODE_UNMERGED = 0, ATMM_MODE_MERGED = 1, ATMM_MODE_MIXTURE = 2 };
typedef struct atmm_model_state atmm_model_state;
int atmm_state_create(atmm_registry* r, void* w, int64_t ldw, int64_t w_layer_stride, int w_dtype,
                      atmm_model_state** out);
void atmm_state_destroy(atmm_model_state* st);
int atmm_state_get(const atmm_model_state* st, int* mode, int32_t* merged_adapter, int64_t* weight_writes);
int atmm_state_merge(atmm_model_state* st, int32_t adapter_id, void* stream);
int atmm_state_unmerge(atmm_model_state* st, int32_t adapter_id, void* stream);
/* init_delora (serving.hpp:24-33) + state.mode = Mixture (acceptance.cpp:131-132):
 * requires the adapter to be the merged one. */
int atmm_state_set_mixture(atmm_model_state* st, int32_t adapter_id);
int atmm_state_mode_switch(atmm_model_state* st, int to_mode, int32_t target_adapter, void* stream,
                           int64_t* launches);

/* ===================================================================== */
/* Plain ATMM GEMM (atmm.hpp:111-154)                                    */
/* ===================================================================== */

/* atmm_multiply_into with host fp32 buffers: c = a . b, fp32-faithful
 * (atmm_gemm_f32: split-bf16 operands on tcgen05, fp32 accumulate and
 * output).  cfg is validated like the reference (ConfigError).  Synchronous. */
int atmm_multiply_host(const float* a, int64_t m, int64_t k, const float* b, int64_t n,
                       float* c, const int32_t cfg[6]);

/* ===================================================================== */
/* fp32-faithful path (the reference's fp32 contract on tensor cores)    */
/* ===================================================================== */
/* The reference computes in fp32 and its tests hold results to 1e-4 *
 * max(1, max|ref|) (acceptance.cpp:62-211).  These entry points keep that
 * contract on the bf16 tensor cores: each fp32 operand is split into three
 * bf16 parts x = h + m + l and every product is ONE tcgen05 GEMM over the
 * K-concatenation of the six partial products hh, hm, mh, hl, lh, mm with
 * fp32 accumulation (dropped terms <= 2^-24 relative: fp32 rounding level).
 * 6x the tensor work of the bf16 path; the bf16 entry points above remain
 * the serving path.  Device pointers, fp32, stream-ordered. */

/* A precise registry also keeps the split images of every adapter's factors
 * (set before the first put; combined slots are not available). */
int atmm_registry_set_precise(atmm_registry* r, int on);
/* C = A . B + beta C (beta 0 or 1), any m, k, n and row strides. */
int atmm_gemm_f32(const float* a, int64_t lda, const float* b, int64_t ldb, float* c, int64_t ldc, int64_t m,
                  int64_t k, int64_t n, float beta, void* stream);
/* run_bypass + residual (batch.hpp:48-81, model.hpp:239-241) on a plan of a
 * precise registry: y[row] += scale * s_a * (x[row] . down_a) . up_a. */
int atmm_bypass_apply_f32(const atmm_plan* p, int64_t layer, const float* x, int64_t ldx, float* y, int64_t ldy,
                          float scale, void* stream);
/* merge / unmerge (model.hpp:144-188): W_l += sign * s_a * down_a . up_a for
 * layers [layer0, layer0 + num_layers) of fp32 W (delta_w_into + add_inplace). */
int atmm_merge_apply_f32(atmm_registry* r, int32_t adapter_id, int64_t layer0, int64_t num_layers, float* w, int64_t ldw,
                         int64_t w_layer_stride, float sign, void* stream);
/* delta_w (model.hpp:130-140) into a device fp32 d_in x d_out matrix. */
int atmm_delta_w_f32(atmm_registry* r, int32_t adapter_id, int64_t layer, float* out, int64_t ldo, void* stream);
/* The stack forward (model.hpp:192-328): cur <- tanh(cur . W_l + sum_i
 * scales[i] * bypass_{plans[i], l}(cur)) for l < num_layers.  No plan =
 * forward_merged; one plan = forward_unmerged; forward_mixture = the guest
 * rows' own plan (+1) and the merged adapter's plan over the same rows (-1)
 * on merged weights.  Plans must come from precise registries with
 * d_in == d_out == d and n rows. */
int atmm_forward_f32(const float* w, int64_t ldw, int64_t w_layer_stride, int64_t num_layers, int64_t n, int64_t d,
                     const float* x, int64_t ldx, float* out, int64_t ldo, const atmm_plan* const* plans,
                     const float* scales, int64_t num_plans, void* stream);

/* Host-buffer forms (synchronous; device staging reused across calls):
 * the stack forward of host fp32 W [L][d][d] / x [n][d] into out, and the
 * in-place all-layer merge (sign +1) / unmerge (-1) of host fp32 W
 * [L][d_in][d_out] -- the address of W never changes (acceptance.cpp:188). */
int atmm_forward_f32_host(const float* w, int64_t num_layers, int64_t n, int64_t d, const float* x, float* out,
                          const atmm_plan* const* plans, const float* scales, int64_t num_plans);
int atmm_merge_f32_host(atmm_registry* r, int32_t adapter_id, float* w, float sign);

/* ===================================================================== */
/* Offline tiling search on B200 (atmm.hpp:188-355)                      */
/* ===================================================================== */

/* A tuning shape: one batch of `segments` segments of `m` rows each, every
 * segment its own adapter of rank `rank`, rows shuffled, at (d_in, d_out).
 * The table key is the fused launch's lookup key (m_bucket(m), d_in, rank),
 * like the reference's shrink lookup (batch.hpp:70). */
typedef struct atmm_tune_shape {
  int64_t m, d_in, rank, d_out, segments;
} atmm_tune_shape;

/* benchmark_config (atmm.hpp:188-216): median device time (ns per apply) of
 * `trials` (>= 3, else ConfigError) trials after one warm-up, the launch
 * forced for every segment.  Each trial flushes L2 (256 MB write), then times
 * back-to-back bf16-Y applies on distinct buffers with CUDA events. */
int atmm_benchmark_launch(int device, const atmm_tune_shape* shape, const int32_t launch[5], int trials,
                          uint64_t seed, int64_t* median_ns);
/* grid_bench_ns (atmm.hpp:229-270): scores[s * num_launches + c] = median of
 * `rounds` round medians, rounds interleaved over the whole grid; failed
 * points score INT64_MAX and are described in `failures` (nullable). */
int atmm_grid_bench_ns(int device, const atmm_tune_shape* shapes, int64_t num_shapes, const int32_t* launches,
                       int64_t num_launches, int trials, int rounds, int64_t* scores, char* failures,
                       size_t failures_cap);
/* tiling_search (atmm.hpp:276-330): per-shape argmin over the candidate
 * launches (ties to the lexicographically smallest {tile_m, cluster, bn,
 * stages, path}), 3 interleaved rounds; the most frequent winner becomes the
 * table default (its launch stored as "default_sm100").  Entries carry the
 * measured ns, the B200 launch ("sm100") and an equivalent reference config. */
int atmm_tiling_search(int device, const atmm_tune_shape* shapes, int64_t num_shapes, const int32_t* launches,
                       int64_t num_launches, int trials, atmm_table** out, char* failures, size_t failures_cap);
/* Host-only selection half of tiling_search over scores[s * num_launches + c]
 * (INT64_MAX = failed): the table tiling_search would build from them. */
int atmm_table_from_scores(const atmm_tune_shape* shapes, int64_t num_shapes, const int32_t* launches,
                           int64_t num_launches, const int64_t* scores, atmm_table** out, char* failures,
                           size_t failures_cap);
/* default_shape_grid (atmm.hpp:341-355) for the bypass at (d_in, d_out):
 * segment rows {8 .. 512} x ranks (NULL/0 = {8, 16, 32, 64, 128}), ~1k-token
 * batches.  Writes up to cap shapes and the total count. */
int atmm_default_shape_grid(int64_t d_in, int64_t d_out, const int64_t* ranks, int64_t num_ranks, atmm_tune_shape* out,
                            int64_t cap, int64_t* count);
/* default_candidates (tiling.hpp:124-149) for B200: the curated launch list
 * (5 ints each). */
int atmm_default_launch_candidates(int32_t* out, int64_t cap, int64_t* count);

/* ===================================================================== */
/* Request sharding over GPUs                         */
/* ===================================================================== */

/* Longest-processing-time partition of the segments of plan_batch(assignment)
 * over num_shards GPUs, cost = rows * rank * (d_in + d_out) + adapter bytes.
 * Writes shard_of_row[n]; whole segments stay together.  Deterministic. */
int atmm_shard_rows(const int32_t* assignment, int64_t n, const int32_t* adapter_ids,
                    const int64_t* adapter_ranks, int64_t num_adapters, int64_t d_in,
                    int64_t d_out, int32_t num_shards, int32_t* shard_of_row);

/* ===================================================================== */
/* Layer forward (model.hpp:192-328)                                      */
/* ===================================================================== */

/* The serving model's stack forward on device, replacing forward_unmerged
 * (model.hpp:216-246), forward_mixture (model.hpp:251-328) and
 * forward_merged (model.hpp:192-211):
 *     cur <- tanh(cur . W_l + bypass_l(cur)),  l = 0 .. num_layers-1
 * bypass_l is the plan's batched LoRA at layer l (run_bypass,
 * batch.hpp:48-81).  A mixture plan (combined slots over the guest rows, see
 * atmm_plan_create_mapped) gives forward_mixture over merged weights; a NULL
 * plan gives forward_merged.  The bypass rides the base GEMM as extra K
 * blocks of the same tcgen05 accumulator; bf16 activations and weights,
 * fp32 accumulation, tanh, bf16 out.
 *
 * create: plan may be NULL (then device, n and hidden_dim give the shape;
 * otherwise they may be 0 or must match the plan).  The forward owns its
 * workspace (two n x d activation buffers, the K-extension images) and
 * references the plan's registry: replacing an adapter makes it stale
 * (ATMM_ERR_CONFIG at run).
 * run: W is num_layers x [d][d] bf16 (row stride ldw, layer stride
 * w_layer_stride elements, the reference's BaseModel layer layout), X and
 * out are n x d bf16 (row strides ldx / ldo, multiples of 8; 16-byte aligned
 * bases; out must not overlap X).  Stream-ordered on `stream`.
 * num_layers = 0 copies X.
 * Concurrency: one forward object is SINGLE-STREAM -- its activation
 * ping-pong buffers and K-extension images are per object, so two runs of
 * the same object must be ordered (same stream, or an event between them).
 * Run concurrent forwards through separate objects (the reference's CPU
 * forward is reentrant; this is the device equivalent of one call frame). */
typedef struct atmm_forward atmm_forward;
int atmm_forward_create(const atmm_plan* plan, int device, int64_t n, int64_t hidden_dim,
                        atmm_forward** out);
/* Explicit tile options of the base GEMM (layer forward and atmm_gemm_ex);
 * a zero field (pair: -1) leaves that choice to the built-in heuristic.
 * Every option combination computes the same product; they exist for tile
 * sweeps and path-coverage tests.  Invalid values -> ATMM_ERR_CONFIG. */
typedef struct atmm_gemm_opts {
  int32_t pair;   /* -1 automatic, 0 1-SM tiles, 1 2-SM CTA pairs (cta_group::2) */
  int32_t bn;     /* N tile: 0 automatic, 128, 256 */
  int32_t kz;     /* 1-SM split-K cluster: 0 automatic, 1, 2, 4, 8 (bn 128 only) */
  int32_t ks;     /* layer forward: shrink K split, 0 automatic, 1..16 */
  int32_t mc;     /* plain GEMM: A multicast over mc N tiles, 0/1 off, 2, 4 */
  int32_t stages; /* GEMM ring depth cap: 0 automatic, 2..8 */
} atmm_gemm_opts;
int atmm_forward_create_opts(const atmm_plan* plan, int device, int64_t n, int64_t hidden_dim,
                             const atmm_gemm_opts* opts, atmm_forward** out);
void atmm_forward_destroy(atmm_forward* f);
int atmm_forward_run(atmm_forward* f, const void* w, int64_t ldw, int64_t w_layer_stride,
                     int64_t num_layers, const void* x, int64_t ldx, void* out, int64_t ldo,
                     void* stream);
/* {n, d, bn, tiles, grid, ext blocks, shrink items, shrink K split, sorted,
 *  GEMM stages, shrink stages, GEMM cta_group (1 or 2), GEMM split-K}: the
 *  first min(cap, 13) are written. */
int atmm_forward_stats(const atmm_forward* f, int64_t* out, int64_t cap);

/* Plain device GEMM C = A . B, the base-model product of every layer
 * (atmm_multiply_into, atmm.hpp:111-154, with a dense right operand as in
 * model.hpp:238): A m x k bf16 row-major (row stride lda), B k x n bf16
 * row-major (ldb), C m x n (ldc) in c_dtype ATMM_BF16 or ATMM_F32, fp32
 * accumulation on the tensor cores, C overwritten.  n a multiple of 8;
 * lda / ldb multiples of 8, ldc 16-byte aligned rows; 16-byte aligned bases.
 * The device is the current one; stream-ordered on `stream`.  k = 0 zeroes C. */
int atmm_gemm(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int c_dtype,
              int64_t m, int64_t k, int64_t n, void* stream);
/* atmm_gemm with explicit tile options (NULL = automatic). */
int atmm_gemm_ex(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int c_dtype,
                 int64_t m, int64_t k, int64_t n, const atmm_gemm_opts* opts, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ATMM_B200_H_ */
