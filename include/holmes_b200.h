/* holmes_b200.h — C ABI of the B200 ensemble-serving hot path.
 *
 * The reference (zooserve, pure Python) has no FFI: its plug points are Python
 * callables.  Each entry point below replaces one of them; the Python mirror in
 * paper_2008_04063_b200/ binds them with ctypes (INTEGRATION.md shows the
 * binding a zooserve maintainer would add).
 *
 *   hb_create / hb_add_member / hb_set_selector
 *       replace the zoo + selector bookkeeping of `_WindowScorer.__init__`
 *       (pkg/src/zooserve/runtime.py:121-129) and `_check_modalities`
 *       (runtime.py:139-147): members are real 1-D ResNets (arch.py), the
 *       selector is the ensemble bitmask (zoo.py:80-136).
 *   hb_ingest
 *       replaces `Aggregator.add` (runtime.py:98-115) for a whole tick of all
 *       (patient, lead) streams at once: samples go into device ring buffers.
 *   hb_tick
 *       replaces `_WindowScorer.draw` (runtime.py:131-136) + `service_time`
 *       (latency.py:145-151): window gather/z-norm, every selected member's
 *       forward, and the ensemble aggregate, for all patients, per tick.
 *   hb_sweep_auc
 *       replaces `exhaustive_search`'s batched accuracy pass
 *       `roc_auc_many(labels, scores @ bits.T / pop)` (composer.py:614-619,
 *       metrics.py:30-76) with exact midrank AUCs.
 *
 * Conventions: every call returns an hb_status; 0 = ok.  Non-zero codes map
 * onto the reference's exception classes (errors.py): HB_E_INVALID ->
 * ValueError, HB_E_CONFIG -> ConfigurationError, HB_E_EMPTY ->
 * EmptyEnsembleError, HB_E_METRIC -> UndefinedMetricError.  The caller owns
 * host buffers; the context owns device memory.  All work is stream-ordered;
 * `stream` is a cudaStream_t passed as void* (NULL = the context's own
 * stream).  A context is not thread-safe (the Python side holds a lock, as
 * the reference's wall-clock mode does around the scorer, runtime.py:367-368).
 * There is no CPU fallback: without a CUDA device every call fails.
 */
#ifndef HOLMES_B200_H
#define HOLMES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HB_OK = 0,
  HB_E_INVALID = 1, /* ValueError */
  HB_E_CONFIG = 2,  /* ConfigurationError */
  HB_E_EMPTY = 3,   /* EmptyEnsembleError */
  HB_E_CUDA = 4,    /* device failure (DeviceError) */
  HB_E_STATE = 5,   /* call order violated */
  HB_E_METRIC = 6   /* UndefinedMetricError */
} hb_status;

typedef struct hb_ctx hb_ctx;

typedef struct {
  int max_patients; /* P: streams are [P][n_leads] */
  int n_leads;      /* ECG leads per patient (3) */
  int fs;           /* sampling rate, Hz (250) */
  int window_len;   /* samples per window (fs * window_s = 7500) */
  int hop;          /* samples appended per tick (250 = 1 s tick; == window_len: tumbling) */
  int ring_len;     /* ring buffer length per stream (>= window_len; 0 = auto) */
  int keep_windows; /* 1 = retain each tick's raw windows for hb_last_windows (diagnostics) */
} hb_config;

int hb_version(void);
/* Last error message of ctx, or of the calling thread's last failed hb_create when ctx is NULL. */
const char* hb_last_error(const hb_ctx* ctx);

int hb_create(int device, const hb_config* cfg, hb_ctx** out);
int hb_destroy(hb_ctx* ctx);

/* Register zoo member `idx` (zoo order) reading lead `lead` (0-based) with the
 * architecture of ModelProfile(width, depth).  `params` is the flat fp32 blob of
 * arch.flatten_params: per conv layer W[cout][cin][16] then bias[cout] (BN
 * folded), in execution order, then fc_w[c_last], fc_b[1].  Weights are
 * converted to fp16 tensor-core operands on the device. */
int hb_add_member(hb_ctx* ctx, int idx, int lead, int width, int depth, const float* params, size_t n_floats);

/* Ensemble selector: bits[n], bit k <-> member idx k.  Members must be registered. */
int hb_set_selector(hb_ctx* ctx, const uint8_t* bits, int n);
/* Number of members the current selector runs (M) and their idx order. */
int hb_selected(const hb_ctx* ctx, int* idx_out, int cap);

/* Append n_per_stream samples [P][n_leads][n_per_stream] (host, fp32) without scoring. */
int hb_ingest(hb_ctx* ctx, const float* samples, int n_per_stream, void* stream);

/* One serving tick: append `hop` new samples per stream from host `samples`
 * ([P][n_leads][hop] fp32; NULL = already staged with hb_stage_device), score
 * the latest window of every patient with every selected member, aggregate.
 * Outputs (host, may be NULL): member_logits[P][M] (selected order),
 * ens_prob[P] = mean of member sigmoids, ens_mean_logit[P] = mean member logit.
 * With host outputs the call synchronises `stream` before returning. */
int hb_tick(hb_ctx* ctx, const float* samples, float* member_logits, float* ens_prob, float* ens_mean_logit,
            void* stream);

/* Pipelined form of hb_tick with host outputs: hb_tick_submit enqueues the
 * tick (H2D of `samples`, the tick graph, one D2H of the outputs into the
 * context's pinned slot `slot` in {0, 1}) and returns; hb_tick_collect waits
 * for that slot and copies the outputs (same meaning as hb_tick's).  A caller
 * may submit tick t+1 before collecting tick t, so the device never idles
 * between ticks on the host round trip.  Submitting into a slot that still
 * holds an uncollected tick -> HB_E_STATE.  Ticks run in submission order on
 * `stream`; use one stream per context. */
int hb_tick_submit(hb_ctx* ctx, const float* samples, int slot, void* stream);
int hb_tick_collect(hb_ctx* ctx, int slot, float* member_logits, float* ens_prob, float* ens_mean_logit);

/* Device-resident variants (benchmarks, zero-copy callers): copy a device
 * buffer [P][n_leads][hop] into the staging area; outputs stay on device. */
int hb_stage_device(hb_ctx* ctx, const float* dev_samples, void* stream);
int hb_tick_device(hb_ctx* ctx, void* stream);
int hb_device_outputs(const hb_ctx* ctx, float** member_logits, float** ens_prob, float** ens_mean_logit);
/* Member-sharded serving (several contexts / GPUs each running a subset of
 * the ensemble): every tick also writes per-patient partial sums
 * sums[2][P] = (sum of member sigmoids, sum of member logits) over this
 * context's members, fixed order.  After a cross-rank SUM reduce,
 * hb_finalize_sums turns them into the ensemble outputs over the total
 * popcount (device pointers, stream-ordered). */
int hb_device_sums(const hb_ctx* ctx, float** sums);
int hb_finalize_sums(const float* sums, int P, int m_total, float* prob, float* logit, void* stream);

/* Device milliseconds of the most recent tick graph (CUDA events on the tick's
 * stream around the graph launch; waits for the tick to finish). */
int hb_last_tick_ms(hb_ctx* ctx, float* ms);
/* Median device milliseconds of `reps` tick-graph launches on the context's
 * stream (after one warm-up launch).  Measures; the stream cursor advances. */
int hb_time_tick(hb_ctx* ctx, int reps, float* median_ms);
/* Build the current selection's tick graphs (if the selection or a member
 * changed) and upload them to the device, without running a tick: a serving
 * loop calls it before its clock starts so the first tick is not charged the
 * one-off plan/capture/instantiate cost (replaces nothing in the reference,
 * whose scorer has no setup, runtime.py:121-129). */
int hb_prepare(hb_ctx* ctx);
/* Diagnostics of the chain launch (K4c, HB_CHAIN=1 with HB_CHAIN_PROF=1 set
 * before the selection is built): per CTA 16 counters of the last tick
 * (producer dependency-wait / weight-wait / stage-wait / total cycles, items,
 * MMA weight-wait / accumulator-wait / stage-wait / total, epilogue
 * accumulator-wait / total).  Returns the grid size (0 = no chain or no
 * profiling), copies min(grid, cap) rows. */
int hb_chain_profile(hb_ctx* ctx, unsigned long long* out, int cap);
/* Timeline of the last chain launch (same switches): per queue item, 5
 * globaltimer ns values (pulled, its weight image in place, its dependencies
 * met, each of its two column halves published), and the items themselves
 * ((layer << 22) | tile).  Returns the item count (0 = off), copies
 * min(count, cap) items. */
int hb_chain_trace(hb_ctx* ctx, unsigned long long* trace, int* items, int cap);

/* Diagnostics: raw gathered windows [P][n_leads][window] (fp32, host) and
 * (mean, std) [P][n_leads][2] of the most recent tick. */
int hb_last_windows(hb_ctx* ctx, float* raw, float* stats, void* stream);
/* Eagerly launch one tick kernel-by-kernel with a CUDA event after every
 * launch (same kernels and order as the graph) and report, per launch: kind
 * (0 ingest/window, 1 stem, 2 tcgen05 conv K4, 3 aggregate + cursor advance,
 * 5 tcgen05 polyphase conv K4b),
 * device milliseconds, algorithmic FLOPs and bytes.  Returns the number of
 * launches (>= 0) or -status.  Advances the stream cursor like a tick. */
int hb_profile_tick(hb_ctx* ctx, void* stream, int cap, int* kinds, float* ms, double* flops, double* bytes);
/* Algorithmic work of one tick: conv FLOPs and activation bytes (all selected members). */
int hb_tick_work(const hb_ctx* ctx, double* flops, double* bytes);
/* Diagnostics: the z-normalised fp16 windows [n_leads][P][window] (IEEE half bit
 * patterns) that the members of the most recent tick consumed (K2's output). */
int hb_last_normalized(hb_ctx* ctx, uint16_t* xn, void* stream);
/* Host-only query of the frozen layer table the library serves (stem first,
 * then conv1/conv2 of every block): per layer 9 ints
 * {cin, cout, stride, lin, lout, pad_left, shortcut (0 none, 1 identity,
 * 2 maxpool), shortcut channels, head}.  Returns the layer count (writes at
 * most cap layers) or -HB_E_INVALID.  No device is touched; the CPU tests
 * compare it with the Python table and the oracle's own restatement. */
int hb_member_layers(int width, int depth, int window, int* out, int cap);

/* ---------------------------------------------------------------- K6 sweep
 * Profiler sweep over a recorded cohort (replaces exhaustive_search's batched
 * accuracy pass `roc_auc_many(labels, scores @ bits.T / pop)`,
 * pkg/src/zooserve/composer.py:614-619, and the accuracy profiler
 * `ensemble_roc_auc`, cohort.py:100-102 / composer.py:301-302).
 * A cohort is scores[N][n] fp64 row-major (caller-owned, copied to the
 * device once) + labels[N] in {0,1}.  AUC = exact Mann-Whitney U from
 * midranks (ties half credit, metrics.py:30-60) of the ensemble mean
 * scores[:, sel].mean(1), summed in fp64 in column order.
 * Errors: labels not 0/1 or non-finite scores -> HB_E_INVALID (ValueError);
 * one class only -> HB_E_METRIC (UndefinedMetricError); an all-zero selector
 * -> HB_E_EMPTY (EmptyEnsembleError). */
typedef struct hb_cohort hb_cohort;
int hb_cohort_create(int device, const double* scores, const int8_t* labels, int N, int n, hb_cohort** out);
int hb_cohort_destroy(hb_cohort* c);
/* Last error of c, or of the calling thread's last failed cohort call when c is NULL. */
const char* hb_cohort_last_error(const hb_cohort* c);
/* Explicit selectors: bits[S][n] (0/1, bit k <-> column k) -> auc_out[S]. */
int hb_cohort_auc(hb_cohort* c, const uint8_t* bits, int S, double* auc_out);
/* Enumerated selectors: values first .. first+count-1 (bit k of the value <->
 * column k, LSB = column 0; n <= 63) -> auc_out[count].  exhaustive_search
 * is (first=1, count=2^n-1), composer.py:615-616. */
int hb_cohort_auc_range(hb_cohort* c, unsigned long long first, long long count, double* auc_out);
/* One selector: the ensemble means ens_out[N] (original row order) and its AUC. */
int hb_cohort_ensemble(hb_cohort* c, const uint8_t* bits, double* ens_out, double* auc_out);
/* One-shot convenience: selectors[S] as 32-bit masks (n <= 32). */
int hb_sweep_auc(int device, const double* scores, const int8_t* labels, int N, int n, const uint32_t* selectors,
                 int S, double* auc_out);

/* ---------------------------------------------------------------- K7 curves
 * Arrival-curve construction for the latency profiler's queueing bound
 * (replaces the quadratic loops of build_arrival_curve, latency.py:198-239).
 * Host buffers in and out; bit-identical to the reference's numpy results.
 *   hb_arrival_widths: widths[c-1] = min_i ts[i+c-1] - ts[i], c = 1..m (ts sorted)
 *   hb_binned_best:    best[k-1]  = max_j csum[j+k] - csum[j], k = 1..n_bins
 *                      (csum has n_bins + 1 entries) */
int hb_arrival_widths(const double* ts, int m, double* widths_out);
int hb_binned_best(const double* csum, int n_bins, double* best_out);
const char* hb_curve_last_error(void);

/* Kernel-level entry points used by the parity tests (device pointers).
 * Activation layouts (fp16, 8-channel groups g, see hb_kernels.cuh):
 *   I: [P][C/8][roundup(L,8)][8];  S: [P][C/8][2][roundup(ceil(L/2),8)][8] (even/odd positions).
 * A stride-1 conv reads I, a stride-2 conv reads S; res is I for res_mode 1
 * (identity), S for res_mode 2 (maxpool(2) of a res_len-long block input);
 * out_split selects the output layout. */
int hb_op_conv1d(const void* in, int P, int cin, int lin, int stride, const float* w_host, const float* b_host,
                 int cout, const void* res, int res_mode, int res_c, int res_len, void* out, int out_split,
                 const float* fc_w_host, float* head_out, void* stream);
/* General form: every layout is Q-phase (hb_kernels.cuh: per 8-channel plane,
 * Q phase sub-planes of roundup(ceil(L/Q), 8) rows, position l at phase l%Q,
 * row l/Q; I = Q1, S = Q2).  kind: 0 = K4 (positions on M; input Q = stride),
 * 1 = K4b polyphase (output phases x channels on M; input Q = stride*128/cout,
 * no fused head), -1 = the serving planner's choice (hb_conv_kind). */
int hb_op_conv1d_q(const void* in, int P, int cin, int lin, int stride, const float* w_host, const float* b_host,
                   int cout, const void* res, int res_mode, int res_c, int res_len, int res_q, void* out, int out_q,
                   const float* fc_w_host, float* head_out, int kind, void* stream);
int hb_conv_kind(int cin, int cout, int stride, int head);
/* Head partials per patient (head_out of hb_op_conv1d_q is [P][this]) for a head layer of `kind`. */
int hb_conv_head_mt(int P, int cin, int cout, int lin, int stride, int res_mode, int kind);
/* M tiles per patient of a conv layer (head_out of hb_op_conv1d is [P][this]). */
int hb_conv_mt(int cin, int cout, int lin, int stride, int head);
/* Micro-benchmark of one conv layer shape on zero data: mean ms per launch. */
int hb_bench_conv(int P, int cin, int cout, int lin, int stride, int res_mode, int iters, float* ms_out);
int hb_bench_conv_k(int P, int cin, int cout, int lin, int stride, int res_mode, int kind, int iters, float* ms_out);
int hb_op_stem(const void* xn, int P, int L, const float* w_host, const float* b_host, int cout, void* out,
               void* stream);
int hb_op_stem_q(const void* xn, int P, int L, const float* w_host, const float* b_host, int cout, void* out,
                 int out_q, void* stream);
/* Micro-benchmark of the stem (K3) on zero data, G members x Pm rows: mean ms per launch. */
int hb_bench_stem(int G, int Pm, int L, int cout, int out_q, int iters, float* ms_out);

#ifdef __cplusplus
}
#endif
#endif
