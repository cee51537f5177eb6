// Internal kernel interfaces shared by the C-ABI layer (hb_api.cu) and the
// kernel translation units.  Activation layout everywhere ("NG8"):
//   act[p][c/8][Lp][8]  fp16,  Lp = roundup(L, 8), rows [L, Lp) kept zero,
// i.e. per patient, one contiguous [Lp x 16 B] plane per 8-channel group.  A
// conv's implicit-GEMM A tile for one 8-channel group is then one contiguous
// run of rows, and a tap shift is a 16-byte shift of the smem descriptor.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <utility>
#include <vector>

namespace hb {

constexpr int kTaps = 16;
constexpr int kBM = 128;               // output positions per tile (UMMA M)
// Epilogue split of a K4b / K4c tile's columns: K4b drains every tile with all
// four epilogue warpgroups (a quarter each: the accumulator is held half as
// long), K4c with the two warpgroups of its accumulator's parity (a half each,
// alternate tiles).  The fused head writes one partial per column QUARTER in
// both, so a bed's head sum has the same fp32 grouping on either path.
constexpr int kEpiPartsPP = 4;
constexpr int kEpiPartsChain = 2;
constexpr int kHeadParts = 4;
constexpr int kConvThreads = 384;      // warp0 TMA, warp1 MMA, warp2 TMEM, warps 4-7 / 8-11 epilogue
constexpr uint32_t kSmemLimit = 232448;  // 227 KB opt-in dynamic smem on sm_100

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Activation layouts (fp16, per patient p and 8-channel group g of G):
//   I  "interleaved":  rows l of a plane of lp_I(L) rows, element ((p*G+g)*lp + l)*8 + c
//   S  "parity-split": two planes of lh_S(L) rows each (even / odd positions),
//                      position l at (((p*G+g)*2 + (l&1))*lh + (l>>1))*8 + c
// Padding rows (positions >= L inside the planes) are always written as zero
// by the producing kernel.  A stride-1 conv reads I; a stride-2 conv reads S
// (so that both parities are contiguous runs of 128-byte TMA lines); the conv
// feeding a stride-2 conv writes S.
inline int lp_I(int L) { return round_up(L, 8); }
inline int lh_S(int L) { return round_up((L + 1) / 2, 8); }
inline int act_rows(int L, int split) { return split ? 2 * lh_S(L) : lp_I(L); }
// General Q-phase layout (Q a power of two; I = Q1, S = Q2): per plane, Q
// phase sub-planes of lq_Q(L, Q) rows; position l at phase l % Q, row l / Q:
//   element (((p*G+g)*Q + l%Q)*lq + l/Q)*8 + c
// The polyphase conv (conv_pp.cu) reads its input with Q = stride * 128/cout.
// Q * lq_Q(L, Q) is the smallest multiple of 8Q >= L, so every Q <= 32 fits in
// roundup(L, 256) rows per plane.
inline int lq_Q(int L, int Q) { return round_up((L + Q - 1) / Q, 8); }
inline int act_rows_q(int L, int Q) { return Q * lq_Q(L, Q); }
inline int ilog2(int q) {
  int s = 0;
  while ((1 << s) < q) ++s;
  return s;
}
__host__ __device__ __forceinline__ size_t q_off(size_t plane, int qs, int lq, int l) {
  return (((plane << qs) + static_cast<size_t>(l & ((1 << qs) - 1))) * static_cast<size_t>(lq) +
          static_cast<size_t>(l >> qs)) * 8;
}

struct ConvArgs {
  int P, cin, cout, bn, n_ntiles;  // P = G*Pm rows of the activation tensors; bn = per-tile N (mult of 16, <=256)
  int G, Pm;                       // members sharing this layer shape (one launch), patients per member
  int fold, bnp, stride_m;         // taps folded into N (D' = [128 x fold*bn]), MMA N, output rows per M tile
  int lin, lout;
  int out_qs, out_lq;              // output layout: Q = 1 << out_qs phases of out_lq rows
  int out_rows;                    // positions that must be written (valid or zero padding)
  int stride, pad, row0;           // row0: first A row (s=1) / pair (s=2) loaded, multiple of 8
  int ck, n_kchunks, rows;         // channels per k-chunk, A rows per (parity, group) region
  int mt_per_p, num_tiles;
  uint32_t a_stage_bytes, b_chunk_bytes;
  int na_stages, nb_slots, b_resident;
  uint32_t tmem_cols;
  const uint8_t* wpack;            // [G][ntile][kchunk][kstep][2][bn][16 B] fp16
  size_t wpack_stride;             // bytes per member
  const float* bias;               // [G][n_ntiles*bn] (zero padded)
  int bias_stride;                 // floats per member
  int sb_len;                      // floats of bias (and of fc) cached in smem: G*bn, 0 = read global
  __half* out;                     // output activation (Q-phase layout out_qs)
  const __half* res;               // shortcut source or null
  int res_mode;                    // 0 none, 1 identity, 2 maxpool(2)
  int res_c, res_qs, res_lq;       // shortcut channels; its layout (1 << res_qs phases of res_lq rows)
  int relu;
  const float* fc_w;               // head: [G][cout] -> head_out[G*Pm][n_ntiles][mt_per_p] (null = no head)
  float* head_out;
  size_t head_g_stride;            // floats between members' head partials (patient-chunked groups)
  int dbg;                         // experiments only (HB_DEBUG env)
  unsigned long long* prof;        // dbg & 8: per-CTA role cycle counters [grid][8]
  int pair;                        // CTA pairs (cta_group::2, M = 256 = two M tiles, B split along N)
  int mtp_per_p;                   // pair mode: M-tile pairs per (member, N tile) (num_tiles counts pairs)
  int half;                        // pair mode with M = 128 over the pair: 64 output rows per CTA
  uint32_t b_slot_bytes;           // B bytes per slot in this CTA (pair mode: half a k-chunk's image)
};

struct ConvPlan {
  ConvArgs args;
  CUtensorMap tmap;                // A operand view of the input activation
  CUtensorMap tmapB;               // pair mode: the packed weight images as 128-B rows
  int grid;
  uint32_t smem_bytes;
};

// K4b polyphase conv (conv_pp.cu): narrow layers, M = (output phase, C_out).
struct PPArgs {
  int G, Pm, P;                    // members of one launch, patients per member, P = G*Pm
  int cin, cout, stride, pad, lin, lout;
  int ph, Q, qs, U;                // output phases 128/cout, input phases stride*ph = 1 << qs, shifts
  int n_pairs;                     // 16-channel K groups (cin / 16)
  int n_res_pairs;                 // identity shortcut on the tensor core: 16-channel groups of x (0 = epilogue)
  uint32_t z_off, z_half_bytes, z_pair_bytes;  // shortcut selection arrays Z in the weight image
  uint32_t w_par16;                // one tap-parity array, 16-B units
  uint32_t w_half_bytes, w_pair_bytes, w_bytes;  // weight image: [pair][half][parity][entry][cout][16 B]
  size_t w_stride;                 // bytes per member image
  int in_lq;                       // input rows per phase plane
  int nb, R;                       // MMA N (columns per tile); rows per phase plane in a B stage
  uint32_t stage_bytes;            // 2 halves x Q phases x R rows x 16 B
  int n_stages;
  int nt_per_p, num_tiles;
  uint32_t tmem_cols;
  const uint8_t* wimg;
  const float* bias;
  int bias_stride;
  __half* out;
  int out_qs, out_lq, out_rows;
  const __half* res;
  int res_mode, res_c, res_qs, res_lq;
  const float* fc_w;               // fused mean-pool.FC head ([G][cout]) instead of an output, or null
  float* head_out;                 // [G][head_g_stride]: per patient head_mt = nt_per_p*8 partials
  size_t head_g_stride;
  int head_mt;
  int member_split;                // CTAs partitioned by group member (no weight reloads inside a CTA)
  int dbg;                         // experiments only (HB_PP_DBG): 1 no epilogue math/stores, 2 no MMAs, 4 no B loads,
                                   // 16 role cycle counters into prof, 32 zero shortcut rows, 64 L2-only shortcut loads
  unsigned long long* prof;        // dbg & 16: per CTA [8]
};
struct PPPlan {
  PPArgs args;
  CUtensorMap tmap;                // input view {8-row lines, lines, Q phases, planes}
  CUtensorMap tmapX;               // shortcut view (same box) when the shortcut runs as MMAs
  int grid;
  uint32_t smem_bytes;
};
// K4c: several member-group chains of K4b layers in one persistent launch
// (conv_pp.cu: chain_pp_kernel).  Layer descriptors are in the parameter
// block, tensor maps in global memory; per-tile counters order producer and
// consumer tiles inside the launch.
constexpr int kChainStages = 8;          // stage barriers (a layer uses its plan's n_stages <= this)
constexpr uint32_t kChainFixed = 1024;   // barriers, item ring, TMEM holder, before the weight image
constexpr int kChainRing = 8;            // items in flight between the producer and the MMA / epilogue roles
constexpr int kMaxChainLayers = 64;  // (the parameter block stays under 17 KB of the 32 KB limit)
struct ChainArgs {
  PPArgs L[kMaxChainLayers];
  int dep_in[kMaxChainLayers];     // chain layer writing this layer's input (-1: written before the launch)
  int dep_res[kMaxChainLayers];    // chain layer writing its shortcut source (-1: none / before the launch)
  int flag_base[kMaxChainLayers];  // first tile counter of the layer
  const CUtensorMap* tmaps;        // [layer][2] (input view, shortcut view), global, 64-B aligned
  const int* items;                // per queue ((chain, member) pair), layer-major: (layer << 22) | tile
  const int* queue_off;            // [n_chains + 1]
  const int* home;                 // [grid]: the queue a CTA drains first
  int n_chains;                    // queues
  unsigned* ctr;                   // [n_chains] queue heads (reset by the last CTA out)
  const int4* idesc;               // per item: {(layer << 22) | tile, bed row, column tile, member}
  const int4* ideps;               // per item: counter index ranges [x, y) (input) and [z, w) (shortcut)
  unsigned* flags;                 // tile counters (+2 per launch: two column halves)
  int opts;                        // HB_CHAIN_OPTS experiment bits
  int stems_flagged;               // the stems publish tile counters: no whole-grid wait on them
  unsigned* sync;                  // [0] finished launches (epoch), [1] CTAs out of the current launch
  unsigned long long* prof;        // HB_CHAIN_PROF: per CTA [16] role cycle counters (null = off)
  unsigned long long* trace;       // HB_CHAIN_PROF: per queue item [5] globaltimer ns: pulled, weights in place,
                                   // dependencies met, column half 0 / 1 published
  // Ensemble aggregation fused into the chain (agg != 0; else K5 runs after it): the warp whose head-tile
  // half completes a bed (per-bed counter reaches bed_target * (epoch + 1)) sums every member's head
  // partials of that bed in K5's order and writes the bed's outputs; the last CTA out advances the ring
  // cursor.  heads is a `const HeadMember*` (declared below).
  int agg;
  int n_heads, P;                  // members (selection order), beds of the tick
  int bed0, n_beds;                // this launch's bed chunk: beds [bed0, bed0 + n_beds) (counters chunk-local)
  const void* heads;
  float* member_logits;            // [P][n_heads]
  float* ens_prob;
  float* ens_logit;
  float* ens_sums;                 // [2][P]
  long long* wpos;
  int advance;
  unsigned* bed_ctr;               // [P], never reset (epoch-relative targets)
  unsigned bed_target;             // head-tile halves per bed per launch
};
struct ChainLayerIn {
  const struct PPPlan* plan;
  int dep_in, dep_res;             // chain layer index, -1 = written before the launch, kChainDepStem = the stem
  int chain;                       // independent sequence (a member group): CTAs are partitioned by chain
};
constexpr int kChainDepStem = -2;
// A chain's stem when it publishes tile counters (launch_stems): its tile grid.
struct ChainStemIn {
  int tiles_per_row, groups_per_blk, out_rows, rows;
};
struct ChainPlan {
  ChainArgs* args = nullptr;       // host copy of the parameter block
  CUtensorMap* d_tmaps = nullptr;
  int* d_items = nullptr;
  int* d_item_off = nullptr;       // queue offsets, then home chains
  unsigned* d_flags = nullptr;
  unsigned* d_sync = nullptr;
  unsigned long long* d_prof = nullptr;
  unsigned long long* d_trace = nullptr;
  unsigned* d_bed = nullptr;       // per-bed head counters (fused aggregation)
  int4* d_idesc = nullptr;
  int4* d_ideps = nullptr;
  std::vector<unsigned*> stem_flags;  // per chain: its stem's tile counters (inside d_flags), when flagged
  int n_items = 0;
  int grid = 0, n_layers = 0;
  uint32_t smem_bytes = 0;
  double flops = 0, bytes = 0;     // algorithmic work per launch (set by the caller)
};
bool pp_shape_ok(int cin, int cout, int stride);
int pp_phases(int cout);           // 128 / cout; the input of a pp conv is in Q = stride * phases layout
// zc > 0: the image also carries the identity-shortcut selection arrays for zc
// shortcut channels (appended; plan_pp uses them when the shortcut's layout allows).
size_t pp_wbytes(int cin, int cout, int stride, int zc = 0);
void pp_pack_weights(const float* w, int cin, int cout, int stride, uint16_t* dst /* fp16 bits */, int zc = 0);
const char* plan_pp(PPPlan* plan, int G, int Pm, int cin, int cout, int lin, int lout, int stride, int pad,
                    const __half* in, __half* out, int out_q, const uint8_t* wimg, const float* bias,
                    const __half* res, int res_mode, int res_c, int res_len, int res_q, int num_sms, int zc = 0,
                    const float* fc_w = nullptr, float* head_out = nullptr, size_t head_g_stride = 0,
                    int prefer_nb = 0 /* column tile to use where it fits (K4c), 0 = the tile model */);
cudaError_t launch_pp(const PPPlan& plan, cudaStream_t st);
// stems: per chain, or null (every stem output is complete before the launch: PDL wait)
const char* plan_chain(ChainPlan* cp, const ChainLayerIn* layers, int n_layers, int num_sms,
                       const ChainStemIn* stems = nullptr);
void free_chain(ChainPlan* cp);
cudaError_t launch_chain(const ChainPlan& cp, cudaStream_t st);
cudaError_t init_pp_kernel();

// Build a plan (tensor map + tiling) for one conv layer.  The input layout is
// I for stride 1 and S for stride 2; res (if any) and the output may use any
// Q-phase layout (res_q, out_q).  Returns 0 or an error string.
// G members of identical layer shape run in one launch: activations are
// [G*Pm] patients deep, weights / bias / fc are G consecutive per-member images.
const char* plan_conv(ConvPlan* plan, int G, int Pm, int cin, int cout, int lin, int lout, int stride, int pad,
                      const __half* in, __half* out, int out_q, const uint8_t* wpack, const float* bias,
                      const __half* res, int res_mode, int res_c, int res_len, int res_q, const float* fc_w,
                      float* head_out, int num_sms, size_t head_g_stride = 0);
size_t bias_len(int cout);  // per-member bias floats (zero padded to whole N tiles)
int conv_fold(int cin, int cout, int stride);  // taps folded into the MMA N dimension (1, 2 or 4)
int conv_stride_m(int fold);                   // output rows per M tile (128, or 120 when folded)
// Programmatic dependent launch on/off (HB_NO_PDL=1 disables).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// Host-side packing of canonical weights W[cout][cin][16] into the plan's B image.
size_t wpack_bytes(int cin, int cout);
void pack_weights(const float* w, int cin, int cout, int stride, uint16_t* dst /* fp16 bits */);
int conv_bn(int cout);
cudaError_t launch_conv(const ConvPlan& plan, cudaStream_t st);
// one-time kernel attribute setup (opt-in shared memory); call before capture.
cudaError_t init_conv_kernel();
cudaError_t init_stream_kernels();
cudaError_t init_stem_kernel();
inline cudaError_t init_kernels() {
  cudaError_t e = init_conv_kernel();
  if (e == cudaSuccess) e = init_pp_kernel();
  return e != cudaSuccess ? e : init_stream_kernels();
}

// stem conv (C_in = 1) + bias + ReLU on tcgen05 (one K=16 MMA per tile) for G members of one
// group: member g reads xn + x_off[g] ([Pm][L] fp16), weights w[g][cout][16],
// b[g][cout]; writes rows [g*Pm, (g+1)*Pm) of the NG8 output.
struct StemMember {
  const __half* x;  // [Pm][x_stride]
  const float* w;   // [cout][16]
  const float* b;   // [cout]
};
constexpr int kMaxGroup = 16;
cudaError_t launch_stem(const StemMember* members /*host array, G entries*/, int G, int x_stride, int Pm, int L,
                        int out_q, int cout, int pad, __half* out, cudaStream_t st);  // out: Q-phase layout
// Several member groups' stems in one launch (one programmatic predecessor for
// the K4c chain), on at most grid_cap CTAs (0 = one per SM).  With `flags` set
// each tile publishes itself (+1 per column half; tile = row * tiles_per_row +
// block * groups_per_block + phase group, row = g * Pm + p): the chain's first
// layers start on published tiles while the stem still runs.
struct StemGroup {
  const StemMember* members;  // host array, G entries
  int G, x_stride, Pm, L, out_q, cout, pad;
  __half* out;
  unsigned* flags;            // tile counters or null
};
cudaError_t launch_stems(const StemGroup* groups, int n, int grid_cap, cudaStream_t st);
// Stem tiles per activation row (1024-position blocks x phase groups); 0 = the builder kernel serves the shape
int stem_tiles_per_row(int L, int out_q, int cout);

// K1+K2: ring append of `n_new` samples per stream at the device write cursor
// *wpos, then (if xn != null) gather of the window ending at *wpos + n_new and
// z-normalisation -> xn[lead][P][window] fp16.  raw_out (optional) receives the
// raw gathered window [P][leads][window] fp32, stats (optional) mean/std.
cudaError_t launch_ingest_window(const float* staged /*[P][leads][n_new]*/,
                                 float* ring /*[P][leads][R + window]: ring + mirror of its first window slots*/,
                                 const long long* wpos, int P, int leads, int n_new, int R, int window,
                                 __half* xn /*[leads][xn_rows][roundup(window, 8)]*/, int xn_rows, float* raw_out,
                                 float* stats, cudaStream_t st);
cudaError_t launch_advance(long long* wpos, int n, cudaStream_t st);

// head + ensemble aggregation: partial[m][P][mt] -> member logits, ensemble outputs.
struct HeadMember {
  const float* partial;  // [P][mt]
  int mt;
  float inv_len;
  float fc_b;
};
cudaError_t launch_aggregate(const HeadMember* members_dev, int M, int P, float* member_logits /*[P][M]*/,
                             float* ens_prob, float* ens_logit, float* ens_sums /*[2][P]*/, long long* wpos /*advanced by `advance`, may be null*/,
                             int advance, cudaStream_t st);
cudaError_t launch_finalize(const float* sums, int P, int m_total, float* prob, float* logit, cudaStream_t st);
constexpr int kMaxMembers = 64;

}  // namespace hb
