// C-ABI layer (include/holmes_b200.h): the serving context, member registry,
// per-tick CUDA graph (ingest/window -> members' stem + tcgen05 convs ->
// aggregate -> cursor advance), and kernel-level test entry points.
#include "../../include/holmes_b200.h"
#include "hb_kernels.cuh"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named host ranges for nsys / ncu --nvtx

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

using namespace hb;

namespace {

thread_local std::string g_create_err;

// RAII NVTX range over a C-ABI call (free when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct LayerSpec {
  int cin, cout, stride, lin, lout, pad, res_mode, res_c, head;
};

// Same table as paper_2008_04063_b200/arch.py:member_layers (stem first).
std::vector<LayerSpec> member_layers(int width, int depth, int window) {
  std::vector<LayerSpec> v;
  auto same = [](int lin, int s, int* lout, int* pad) {
    *lout = (lin + s - 1) / s;
    const int tot = (*lout - 1) * s + kTaps - lin;
    *pad = tot > 0 ? tot / 2 : 0;
  };
  int lo, pd;
  same(window, 1, &lo, &pd);
  v.push_back({1, width, 1, window, lo, pd, 0, 0, 0});
  int len = window;
  for (int i = 0; i < depth; ++i) {
    const int s = (i % 2 == 1) ? 2 : 1;
    const int cin = (i == 0) ? width : width * (1 << ((i - 1) / 4));
    const int cout = (i % 4 == 0 && i > 0) ? 2 * cin : cin;
    int l1, p1, l2, p2;
    same(len, s, &l1, &p1);
    same(l1, 1, &l2, &p2);
    v.push_back({cin, cout, s, len, l1, p1, 0, 0, 0});
    v.push_back({cout, cout, 1, l1, l2, p2, s == 2 ? 2 : 1, cin, i == depth - 1 ? 1 : 0});
    len = l2;
  }
  return v;
}

// Conv kernel per layer: K4 (positions on M, conv_tc.cu) or K4b (output
// phases x channels on M, conv_pp.cu) for the narrow layers it supports.
// Measured per shape (profiles/r01_convbench_pp.txt) K4b wins 1.2-2.4x on
// every supported shape at 1024 beds; at 64 beds it loses a few percent on
// some small 64-channel launches in isolation, but inside the two-branch tick
// graph sending every supported layer to K4b is fastest (c2 0.947 vs 0.958 ms
// with a size rule, profiles/r01_pp_ab.txt).  HB_PP=0 keeps every layer on K4.
enum { KIND_TC = 0, KIND_PP = 1 };
bool pp_eligible(const LayerSpec& L) {
  static const bool heads = !(getenv("HB_PP_HEAD") && atoi(getenv("HB_PP_HEAD")) == 0);
  return (heads || !L.head) && L.cin >= 16 && pp_shape_ok(L.cin, L.cout, L.stride);
}
// Head partials per patient of a K4b head layer (nt_per_p * 4 * kEpiParts), from a dry-run plan.
int pp_head_mt(const LayerSpec& L, int G, int Pm, int sms, int prefer_nb = 0) {
  PPPlan plan;
  __half* fake = reinterpret_cast<__half*>(static_cast<uintptr_t>(1) << 20);  // encoded, never dereferenced
  const char* e = plan_pp(&plan, G, Pm, L.cin, L.cout, L.lin, L.lout, L.stride, L.pad, fake, nullptr, 1,
                          reinterpret_cast<uint8_t*>(fake), nullptr, L.res_mode ? fake : nullptr, L.res_mode, L.res_c,
                          L.res_mode == 2 ? 2 * L.lout : L.lout, L.res_mode == 2 ? 2 : 1, sms, 0,
                          reinterpret_cast<const float*>(fake), reinterpret_cast<float*>(fake), 0, prefer_nb);
  return e ? -1 : plan.args.head_mt;
}
// Column tile of every K4c layer where it fits (HB_CHAIN_NB overrides): in one
// persistent launch there are no per-layer waves to quantise, and the widest
// tile measured fastest (tools/abtick.py: 256 vs the per-launch tile model -2 %,
// vs 240 -0.4 %).
int chain_nb() { return getenv("HB_CHAIN_NB") ? atoi(getenv("HB_CHAIN_NB")) : 256; }
int layer_kind(const LayerSpec& L) {
  static const int pp_on = getenv("HB_PP") ? atoi(getenv("HB_PP")) : 1;
  return (pp_on && pp_eligible(L)) ? KIND_PP : KIND_TC;
}
// Input layout (phases Q) a conv of `kind` reads: K4 reads I (s=1) / S (s=2).
int layer_in_q(const LayerSpec& L, int kind) { return kind == KIND_PP ? L.stride * pp_phases(L.cout) : L.stride; }
// K4b images of identity-shortcut layers also carry the shortcut selection
// arrays (the shortcut then runs as MMAs when x's layout allows, conv_pp.cu).
int layer_zc(const LayerSpec& L) { return (L.res_mode == 1 && L.res_c % 16 == 0 && L.res_c <= L.cout) ? L.res_c : 0; }
size_t layer_wbytes(const LayerSpec& L, int kind) {
  return kind == KIND_PP ? pp_wbytes(L.cin, L.cout, L.stride, layer_zc(L)) : wpack_bytes(L.cin, L.cout);
}
void layer_pack(const LayerSpec& L, int kind, const float* w, uint16_t* dst) {
  if (kind == KIND_PP) pp_pack_weights(w, L.cin, L.cout, L.stride, dst, layer_zc(L));
  else pack_weights(w, L.cin, L.cout, L.stride, dst);
}
// Rows per activation plane that hold any Q-phase layout (Q <= 32) of length L.
int plane_rows_max(int L) { return round_up(L, 256); }

struct LayerPlan {
  int kind = KIND_TC;
  ConvPlan tc;
  PPPlan pp;
};
cudaError_t launch_layer(const LayerPlan& lp, cudaStream_t st) {
  return lp.kind == KIND_PP ? launch_pp(lp.pp, st) : launch_conv(lp.tc, st);
}

struct Group {
  int width = 0, depth = 0, lead_any = 0, lane = 0;
  std::vector<int> mi;                 // positions in hb_ctx::selected (zoo order)
  std::vector<LayerSpec> layers;
  std::vector<int> kind;               // per layer (index 0 = stem, unused)
  std::vector<std::vector<StemMember>> stem;  // [chunk][member]: its lead's windows (chunk rows), stem weights
  std::vector<uint8_t*> wpack;         // per conv layer: [G][member image]
  std::vector<float*> bias;            // per conv layer: [G][bias_len]
  float* fc_w = nullptr;               // [G][c_last]
  float* head_partial = nullptr;       // [G*P][mt]
  int head_mt = 0;
  double flops = 0;
  std::vector<size_t> plan0;           // first plan index, per patient chunk
  std::vector<__half*> cbuf;           // chain mode: output of every layer (0 = stem), one buffer each
};

struct Member {
  int idx = -1, lead = 0, width = 0, depth = 0;
  std::vector<LayerSpec> layers;
  std::vector<uint8_t*> wpp;    // per conv layer: K4b weight image (null if not eligible)
  float* stem_w = nullptr;  // [w][16]
  float* stem_b = nullptr;
  std::vector<uint8_t*> wpack;  // per conv layer (layers[1..])
  std::vector<float*> bias;
  float* fc_w = nullptr;
  float fc_b = 0.f;
  int head_mt = 0;
  double flops = 0, bytes = 0;
};

}  // namespace

struct hb_ctx {
  int device = 0, P = 0, leads = 0, fs = 0, W = 0, hop = 0, R = 0, keep = 0, num_sms = 148;
  int max_lanes = 4;  // concurrent member branches in the tick graph (HB_LANES overrides)
  int group_off = 0;  // HB_NO_GROUP=1: one launch per member and layer (A/B experiments)
  int max_group = kMaxGroup;  // HB_MAX_GROUP: cap on members per grouped launch (A/B experiments)
  // patient micro-batching: member chains run over chunks of Pc beds so the
  // activation buffers stay within act_budget (the rings / windows hold all P)
  int Pc = 0, n_chunks = 1, P_pad = 0;
  int chain_pc = 0;                    // beds per K4c launch (chain mode)
  double act_budget = 64e9;
  cudaStream_t own = nullptr;
  float* ring = nullptr;
  float* staged = nullptr;   // [P][leads][hop]: the buffer the tick graph being captured reads
  float* staged_io[2] = {nullptr, nullptr};  // per submit slot (staged_io[0] == the default staged)
  cudaStream_t copy = nullptr;               // submit's H2D runs here, overlapping the previous tick
  cudaEvent_t h2d_done[2] = {nullptr, nullptr};
  float* prefill = nullptr;  // [P][leads][R]
  long long* wpos = nullptr;
  __half* xn = nullptr;      // [leads][P][W]
  float* raw = nullptr;      // [P][leads][W] (keep_windows)
  float* stats = nullptr;    // [P][leads][2]
  std::map<int, Member> members;
  std::vector<int> selected;
  // per-selection resources: selected members of identical architecture form
  // a group that runs as ONE launch per layer (activations G*P patients deep);
  // groups are spread over `lanes` concurrent graph branches, 3 rotating
  // activation buffers per lane (groups on one branch run back to back)
  int lanes = 1;
  std::vector<__half*> act;
  std::vector<Group> groups;
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> ev;
  size_t act_bytes = 0;
  HeadMember* d_heads = nullptr;
  float* member_logits = nullptr;
  float* ens_prob = nullptr;
  float* ens_logit = nullptr;
  float* ens_sums = nullptr;  // [2][P]: sum of member sigmoids, sum of member logits
  // member_logits [P][M], ens_prob [P], ens_logit [P] are one device block;
  // graph_io[s] = the tick graph + one D2H of that block into pinned h_out[s];
  // two slots let a caller submit tick t+1 before collecting tick t
  float* h_out[2] = {nullptr, nullptr};
  cudaGraphExec_t graph_io[2] = {nullptr, nullptr};
  cudaEvent_t io_done[2] = {nullptr, nullptr};
  bool io_busy[2] = {false, false};
  int slot_M[2] = {0, 0};  // members of the tick submitted into each slot (its h_out layout)
  std::vector<LayerPlan> plans;
  // K4c chain mode (default; HB_CHAIN=0 disables): every group's K4b layers in one persistent launch
  // with tile-level dependencies; each layer writes its own buffer (no reuse
  // inside a tick, so no write-after-read hazard between tiles)
  bool chain_on = false;
  int stem_sms = 0;  // chain mode: CTAs of the stem launch (0 = one per SM); the chain takes the other SMs first
  ChainPlan chain;                    // K4c over bed chunk 0 (the only chunk up to HB_CHAIN_MAX_P beds)
  std::vector<ChainPlan> chain_rest;  // K4c over bed chunks 1.. (bed counts above HB_CHAIN_MAX_P)
  cudaGraphExec_t graph = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // bracket the last tick graph launch
  bool timed = false;
  bool dirty = true;
  std::string err;
};

namespace {

int fail(hb_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg; else g_create_err = msg;
  return code;
}

#define CK(c, expr)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) return fail(c, HB_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

cudaStream_t pick(hb_ctx* c, void* s) { return s ? static_cast<cudaStream_t>(s) : c->own; }

void free_selection(hb_ctx* c) {
  if (c->graph) cudaGraphExecDestroy(c->graph);
  c->graph = nullptr;
  for (int k = 0; k < 2; ++k) {
    if (c->graph_io[k]) cudaGraphExecDestroy(c->graph_io[k]);
    c->graph_io[k] = nullptr;
    if (c->h_out[k]) cudaFreeHost(c->h_out[k]);
    c->h_out[k] = nullptr;
    c->io_busy[k] = false;
  }
  for (auto& a : c->act) cudaFree(a);
  c->act.clear();
  free_chain(&c->chain);
  for (auto& cp : c->chain_rest) free_chain(&cp);
  c->chain_rest.clear();
  c->chain_on = false;
  for (auto& g : c->groups) {
    for (auto p : g.cbuf) cudaFree(p);
    for (auto p : g.wpack) cudaFree(p);
    for (auto p : g.bias) cudaFree(p);
    cudaFree(g.fc_w);
    cudaFree(g.head_partial);
  }
  c->groups.clear();
  cudaFree(c->xn);
  c->xn = nullptr;
  for (auto s2 : c->side) cudaStreamDestroy(s2);
  c->side.clear();
  for (auto e : c->ev) cudaEventDestroy(e);
  c->ev.clear();
  c->act_bytes = 0;
  if (c->d_heads) cudaFree(c->d_heads);
  if (c->member_logits) cudaFree(c->member_logits);  // (ens_prob / ens_logit live in the same block)
  if (c->ens_sums) cudaFree(c->ens_sums);
  c->d_heads = nullptr;
  c->member_logits = c->ens_prob = c->ens_logit = c->ens_sums = nullptr;
  c->plans.clear();
}

void free_member(Member& m) {
  cudaFree(m.stem_w);
  cudaFree(m.stem_b);
  for (auto p : m.wpack) cudaFree(p);
  for (auto p : m.wpp) cudaFree(p);
  for (auto p : m.bias) cudaFree(p);
  cudaFree(m.fc_w);
}

// Kernel kinds reported by hb_profile_tick.
enum { K_INGEST = 0, K_STEM = 1, K_CONV = 2, K_AGG = 3, K_ADV = 4, K_CONV_PP = 5, K_CHAIN = 6 };

struct ProfRec {
  std::vector<cudaEvent_t>* ev = nullptr;  // event recorded after every launch
  std::vector<int> kind;
  std::vector<double> flops, bytes;
  void mark(cudaStream_t st, int k, double f, double b) {
    if (!ev) return;
    static const bool dbg_sync = getenv("HB_DEBUG_SYNC") != nullptr;
    if (dbg_sync) {
      fprintf(stderr, "[hb] launch %zu kind %d ...", kind.size(), k);
      const cudaError_t e = cudaStreamSynchronize(st);
      fprintf(stderr, " %s\n", cudaGetErrorString(e));
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev->push_back(e);
    kind.push_back(k);
    flops.push_back(f);
    bytes.push_back(b);
  }
};

// Enqueue the whole tick (after staging) on stream st.
int enqueue_tick(hb_ctx* c, cudaStream_t st, ProfRec* pr = nullptr) {
  ProfRec none;
  if (!pr) pr = &none;
  const double P = c->P;
  CK(c, launch_ingest_window(c->staged, c->ring, c->wpos, c->P, c->leads, c->hop, c->R, c->W, c->xn, c->P_pad,
                             c->keep ? c->raw : nullptr, c->stats, st));
  pr->mark(st, K_INGEST, 0.0, P * c->leads * (c->hop * 8.0 + c->W * 6.0));
  // Members fork into `lanes` branches after the window kernel and join before
  // the aggregate (captured as parallel graph branches).  The eager profiling
  // path (pr->ev set) keeps everything on one stream so per-kernel event times
  // stay clean.
  for (int ch = 0; c->chain_on && ch < c->n_chunks; ++ch) {
    // every group's stem in one launch, then every group's conv chain in one launch, per bed chunk
    const ChainPlan& cp = ch == 0 ? c->chain : c->chain_rest[ch - 1];
    std::vector<StemGroup> sg;
    for (size_t gi = 0; gi < c->groups.size(); ++gi) {
      const Group& g = c->groups[gi];
      const LayerSpec& s0 = g.layers[0];
      sg.push_back({g.stem[ch].data(), static_cast<int>(g.mi.size()), round_up(c->W, 8), c->Pc, c->W,
                    layer_in_q(g.layers[1], g.kind[1]), s0.cout, s0.pad, g.cbuf[0],
                    cp.stem_flags.empty() ? nullptr : cp.stem_flags[gi]});
    }
    // one launch for every group's stem, in the graph and in the eager profile alike
    CK(c, launch_stems(sg.data(), static_cast<int>(sg.size()), c->stem_sms, st));
    {
      double fl = 0, by = 0;
      for (const Group& g : c->groups) {
        const LayerSpec& s0 = g.layers[0];
        const double rows = static_cast<double>(c->Pc) * g.mi.size();
        fl += rows * 2.0 * s0.cout * kTaps * s0.lout;
        by += rows * (2.0 * s0.lin + 2.0 * s0.cout * s0.lout);
      }
      pr->mark(st, K_STEM, fl, by);
    }
    CK(c, launch_chain(cp, st));
    pr->mark(st, K_CHAIN, cp.flops, cp.bytes);
  }
  const bool fork = !c->chain_on && (pr->ev == nullptr) && c->lanes > 1;
  if (fork) CK(c, cudaEventRecord(c->ev[0], st));
  std::vector<bool> lane_started(c->lanes, false);
  for (const Group& g : c->groups) {
    if (c->chain_on) break;
    const int ln = g.lane;
    cudaStream_t ms = fork ? c->side[ln] : st;
    if (fork && !lane_started[ln]) {
      CK(c, cudaStreamWaitEvent(ms, c->ev[0], 0));
      lane_started[ln] = true;
    }
    const int G = static_cast<int>(g.mi.size());
    const double rows = static_cast<double>(c->Pc) * G;
    const LayerSpec& s0 = g.layers[0];
    for (int ch = 0; ch < c->n_chunks; ++ch) {
      CK(c, launch_stem(g.stem[ch].data(), G, round_up(c->W, 8), c->Pc, c->W, layer_in_q(g.layers[1], g.kind[1]), s0.cout,
                        s0.pad, c->act[3 * ln], ms));
      pr->mark(ms, K_STEM, rows * 2.0 * s0.cout * kTaps * s0.lout, rows * (2.0 * s0.lin + 2.0 * s0.cout * s0.lout));
      size_t pi = g.plan0[ch];
      for (size_t li = 1; li < g.layers.size(); ++li) {
        const LayerSpec& L = g.layers[li];
        const int kk = c->plans[pi].kind == KIND_PP ? K_CONV_PP : K_CONV;
        CK(c, launch_layer(c->plans[pi++], ms));
        pr->mark(ms, kk, rows * 2.0 * L.cin * L.cout * kTaps * L.lout,
                 rows * 2.0 * (static_cast<double>(L.cin) * L.lin +
                               (L.head ? 0.0 : static_cast<double>(L.cout) * L.lout) +
                               (L.res_mode ? static_cast<double>(L.res_c) * L.lin : 0.0)));
      }
    }
  }
  if (fork) {
    for (int ln = 0; ln < c->lanes; ++ln) {
      if (!lane_started[ln]) continue;
      CK(c, cudaEventRecord(c->ev[1 + ln], c->side[ln]));
      CK(c, cudaStreamWaitEvent(st, c->ev[1 + ln], 0));
    }
  }
  if (c->chain_on && c->chain.args->agg) return HB_OK;  // aggregation and cursor advance fused into K4c
  CK(c, launch_aggregate(c->d_heads, static_cast<int>(c->selected.size()), c->P, c->member_logits, c->ens_prob,
                         c->ens_logit, c->ens_sums, c->wpos, c->hop, st));
  {  // algorithmic bytes: every member's head partials in, member logits + 2 ensemble outputs + 2 sums out
    double partials = 0.0;
    for (const Group& g : c->groups) partials += static_cast<double>(g.mi.size()) * g.head_mt;
    const double M = static_cast<double>(c->selected.size());
    pr->mark(st, K_AGG, 0.0, P * 4.0 * (partials + M + 4.0));  // (the cursor advance, K_ADV, is fused in)
  }
  return HB_OK;
}

int build_selection(hb_ctx* c) {
  if (!c->dirty) return HB_OK;
  NvtxRange nv("hb:build_selection");
  free_selection(c);
  if (c->selected.empty()) return fail(c, HB_E_EMPTY, "cannot serve an empty ensemble");
  const int M = static_cast<int>(c->selected.size());
  // group selected members by architecture (first-occurrence order; <= kMaxGroup per group)
  for (int mi = 0; mi < M; ++mi) {
    const Member& m = c->members[c->selected[mi]];
    Group* gp = nullptr;
    if (!c->group_off)
      for (auto& g : c->groups)
        if (g.width == m.width && g.depth == m.depth && static_cast<int>(g.mi.size()) < c->max_group) gp = &g;
    if (!gp) {
      c->groups.emplace_back();
      gp = &c->groups.back();
      gp->width = m.width;
      gp->depth = m.depth;
      gp->layers = m.layers;
      gp->kind.assign(gp->layers.size(), KIND_TC);
    }
    gp->mi.push_back(mi);
    gp->flops += m.flops;
  }
  c->lanes = std::max(1, std::min(static_cast<int>(c->groups.size()), c->max_lanes));
  {  // greedy FLOP balance of groups over lanes, largest first
    std::vector<size_t> order(c->groups.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return c->groups[a].flops > c->groups[b].flops; });
    std::vector<double> load(c->lanes, 0.0);
    for (size_t i : order) {
      const int ln = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
      c->groups[i].lane = ln;
      load[ln] += c->groups[i].flops;
    }
  }
  // activation buffers per lane, sized for the largest layer of its groups at
  // Pc beds; Pc halves until 3 rotating buffers per lane fit the budget
  std::vector<size_t> need(c->lanes, 0);
  auto size_for = [&](int pc) {
    std::fill(need.begin(), need.end(), 0);
    for (auto& g : c->groups)
      for (auto& L : g.layers)
        need[g.lane] = std::max(need[g.lane], static_cast<size_t>(pc) * g.mi.size() * L.cout *
                                                  plane_rows_max(L.lout) * sizeof(__half));
    double tot = 0;
    for (size_t v : need) tot += 3.0 * v;
    return tot;
  };
  for (auto& g : c->groups)
    for (size_t li = 1; li < g.layers.size(); ++li) g.kind[li] = layer_kind(g.layers[li]);
  {  // K4c chain mode: every conv of every group on K4b, one patient chunk, each layer its own buffer
    // HB_CHAIN=1 / 0 forces the chain / the per-layer launches (read per build, so tests can
    // switch it); unset, the chain serves bed counts where it measured faster: 8-128 beds
    // (tools/abtick.py, c2: 16 beds 0.243 vs 0.272 ms, 64 beds 0.632 vs 0.693, 128 beds even;
    // 4 beds 0.205 vs 0.156 and 192+ beds slower -- too few tiles per layer to fill a
    // persistent grid, or enough that per-layer launches amortise their fixed costs).
    // The per-launch debug knobs (HB_PP_DBG) exist only on the per-layer path.
    const char* ce = getenv("HB_CHAIN");
    const char* dbg = getenv("HB_PP_DBG");
    const int chain_mode = ce ? atoi(ce) : -1;
    const int min_p = getenv("HB_CHAIN_MIN_P") ? atoi(getenv("HB_CHAIN_MIN_P")) : 8;
    const int max_p = getenv("HB_CHAIN_MAX_P") ? atoi(getenv("HB_CHAIN_MAX_P")) : 128;
    bool ok = chain_mode != 0 && !(dbg && atoi(dbg)) && (chain_mode > 0 || (c->P >= min_p && c->P <= max_p));
    double bytes = 0;
    int n_layers = 0;
    for (auto& g : c->groups)
      for (size_t li = 0; li < g.layers.size(); ++li) {
        const LayerSpec& L = g.layers[li];
        if (li > 0) {
          ok = ok && g.kind[li] == KIND_PP;
          ++n_layers;
        }
        if (!L.head) bytes += static_cast<double>(c->P) * g.mi.size() * L.cout * plane_rows_max(L.lout) * sizeof(__half);
      }
    // HB_CHAIN_CHUNK_P=n: above HB_CHAIN_MAX_P beds run the chain over bed chunks of n (one chain
    // launch per chunk, buffers reused).  Default 0 (off): measured slower than the per-layer
    // launches at every bed count tried (tools/gpu_chunkchain.sh, abtick: 1024 beds 9.38 ms per-layer
    // vs 10.12 / 10.67 / 10.31 ms in chunks of 64 / 96 / 128 and 9.96 ms as one launch; 192-512 alike)
    const int chunk_p = getenv("HB_CHAIN_CHUNK_P") ? atoi(getenv("HB_CHAIN_CHUNK_P")) : 0;
    const bool chunked = chunk_p > 0 && c->P > max_p && chunk_p < c->P;
    ok = ok || (chain_mode < 0 && chunked && !(dbg && atoi(dbg)) && c->P >= min_p);
    for (auto& g : c->groups)
      for (size_t li = 1; li < g.layers.size(); ++li) ok = ok && g.kind[li] == KIND_PP;
    c->chain_on = ok && n_layers <= kMaxChainLayers && bytes * (chunked ? double(chunk_p) / c->P : 1.0) <= c->act_budget;
    c->chain_pc = c->chain_on && chunked ? chunk_p : c->P;
  }
  c->Pc = c->chain_on ? c->chain_pc : c->P;
  while (!c->chain_on && c->Pc > 1 && size_for(c->Pc) > c->act_budget) c->Pc = (c->Pc + 1) / 2;
  size_for(c->Pc);
  c->n_chunks = (c->P + c->Pc - 1) / c->Pc;
  c->P_pad = c->n_chunks * c->Pc;
  {  // normalised windows [leads][P_pad][W]; rows past P stay zero (padding beds of the last chunk)
    const size_t xb = static_cast<size_t>(c->leads) * c->P_pad * round_up(c->W, 8) * sizeof(__half);
    CK(c, cudaMalloc(&c->xn, xb));
    CK(c, cudaMemset(c->xn, 0, xb));
  }
  c->act.assign(3 * c->lanes, nullptr);
  for (int ln = 0; ln < c->lanes && !c->chain_on; ++ln)
    for (int k = 0; k < 3; ++k) {
      CK(c, cudaMalloc(&c->act[3 * ln + k], need[ln]));
      CK(c, cudaMemset(c->act[3 * ln + k], 0, need[ln]));
      c->act_bytes += need[ln];
    }
  c->side.resize(c->lanes);
  for (auto& s2 : c->side) CK(c, cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  c->ev.resize(1 + c->lanes);
  for (auto& e : c->ev) CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const size_t out_floats = static_cast<size_t>(c->P) * (M + 2);
  CK(c, cudaMalloc(&c->member_logits, sizeof(float) * out_floats));
  c->ens_prob = c->member_logits + static_cast<size_t>(c->P) * M;
  c->ens_logit = c->ens_prob + c->P;
  for (int k = 0; k < 2; ++k) CK(c, cudaHostAlloc(&c->h_out[k], sizeof(float) * out_floats, cudaHostAllocDefault));
  CK(c, cudaMalloc(&c->ens_sums, sizeof(float) * 2 * c->P));
  std::vector<HeadMember> heads(M);
  for (auto& g : c->groups) {
    const int G = static_cast<int>(g.mi.size());
    const int c_last = g.layers.back().cout;
    if (c->chain_on)
      for (size_t li = 0; li + 1 < g.layers.size(); ++li) {
        const LayerSpec& L = g.layers[li];
        const size_t b = static_cast<size_t>(c->Pc) * G * L.cout * plane_rows_max(L.lout) * sizeof(__half);
        __half* p = nullptr;
        CK(c, cudaMalloc(&p, b));
        CK(c, cudaMemset(p, 0, b));
        g.cbuf.push_back(p);
        c->act_bytes += b;
      }
    // group-contiguous weight images (device-to-device from the registered members)
    for (size_t li = 1; li < g.layers.size(); ++li) {
      const LayerSpec& L = g.layers[li];
      const size_t wb = layer_wbytes(L, g.kind[li]), bl = bias_len(L.cout);
      uint8_t* w;
      float* b;
      CK(c, cudaMalloc(&w, wb * G));
      CK(c, cudaMalloc(&b, sizeof(float) * bl * G));
      for (int k = 0; k < G; ++k) {
        const Member& m = c->members[c->selected[g.mi[k]]];
        CK(c, cudaMemcpy(w + wb * k, g.kind[li] == KIND_PP ? m.wpp[li - 1] : m.wpack[li - 1], wb,
                         cudaMemcpyDeviceToDevice));
        CK(c, cudaMemcpy(b + bl * k, m.bias[li - 1], sizeof(float) * bl, cudaMemcpyDeviceToDevice));
      }
      g.wpack.push_back(w);
      g.bias.push_back(b);
    }
    CK(c, cudaMalloc(&g.fc_w, sizeof(float) * c_last * G));
    {  // head partials per patient of the last layer, as that layer is tiled
      const LayerSpec& H = g.layers.back();
      if (g.kind.back() == KIND_PP) {
        g.head_mt = pp_head_mt(H, G, c->Pc, c->num_sms);  // (the head's tile width is shape-only in both paths)
        if (g.head_mt <= 0) return fail(c, HB_E_INVALID, "conv_pp: head layer does not plan");
      } else {
        const int bn = conv_bn(H.cout), sm = conv_stride_m(conv_fold(H.cin, H.cout, H.stride));
        g.head_mt = ((round_up(H.cout, 16) + bn - 1) / bn) * ((H.lout + sm - 1) / sm);
      }
    }
    CK(c, cudaMalloc(&g.head_partial, sizeof(float) * G * c->P_pad * g.head_mt));
    g.stem.assign(c->n_chunks, {});
    for (int k = 0; k < G; ++k) {
      const Member& m = c->members[c->selected[g.mi[k]]];
      CK(c, cudaMemcpy(g.fc_w + c_last * k, m.fc_w, sizeof(float) * c_last, cudaMemcpyDeviceToDevice));
      for (int ch = 0; ch < c->n_chunks; ++ch)
        g.stem[ch].push_back(
            {c->xn + (static_cast<size_t>(m.lead) * c->P_pad + static_cast<size_t>(ch) * c->Pc) * round_up(c->W, 8),
             m.stem_w,
             m.stem_b});
      heads[g.mi[k]] = {g.head_partial + static_cast<size_t>(k) * c->P_pad * g.head_mt, g.head_mt,
                        1.f / static_cast<float>(g.layers.back().lout), m.fc_b};
    }
    __half* const* act = &c->act[3 * g.lane];
    for (int ch = 0; ch < c->n_chunks; ++ch) {
      g.plan0.push_back(c->plans.size());
      int cur = 0;
      auto in_q = [&](size_t li) { return layer_in_q(g.layers[li], g.kind[li]); };
      for (size_t li = 1; li < g.layers.size(); ++li) {
        const LayerSpec& L = g.layers[li];
        const bool conv1 = (li % 2 == 1);
        int src = cur, dst, out_q = 1, res_len = 0, res_q = 1;
        const __half* res = nullptr;
        if (conv1) {
          dst = (cur + 1) % 3;
          out_q = in_q(li + 1);  // h feeds conv2
        } else {
          src = (cur + 1) % 3;
          dst = (cur + 2) % 3;
          res = c->chain_on ? g.cbuf[li - 2] : act[cur];
          res_len = g.layers[li - 1].lin;
          res_q = in_q(li - 1);  // the block input, as conv1 read it
          // the block output feeds the next block's conv1 in the layout that conv reads
          out_q = (li + 1 < g.layers.size()) ? in_q(li + 1) : 1;
        }
        const __half* in_buf = c->chain_on ? g.cbuf[li - 1] : act[src];
        __half* out_buf = L.head ? nullptr : (c->chain_on ? g.cbuf[li] : act[dst]);
        // head partials of chunk ch: rows [ch*Pc, (ch+1)*Pc) of every member's [P_pad][head_mt] block
        float* head_base = L.head ? g.head_partial + static_cast<size_t>(ch) * c->Pc * g.head_mt : nullptr;
        LayerPlan plan;
        plan.kind = g.kind[li];
        // HB_LANE_SMS="a,b,..": cap the grid of lane k's conv launches (SM partition experiment)
        int lane_sms = c->num_sms;
        if (const char* ls = getenv("HB_LANE_SMS")) {
          int k = 0;
          for (const char* q = ls; *q; ++k) {
            const int v = atoi(q);
            if (k == g.lane && v > 0) lane_sms = std::min(v, c->num_sms);
            while (*q && *q != ',') ++q;
            if (*q == ',') ++q;
          }
        }
        const char* e;
        if (plan.kind == KIND_PP) {
          e = plan_pp(&plan.pp, G, c->Pc, L.cin, L.cout, L.lin, L.lout, L.stride, L.pad, in_buf,
                      out_buf, out_q, g.wpack[li - 1], g.bias[li - 1], res,
                      conv1 ? 0 : L.res_mode, L.res_c, res_len, res_q, lane_sms, layer_zc(L),
                      L.head ? g.fc_w : nullptr, head_base, static_cast<size_t>(c->P_pad) * g.head_mt,
                      c->chain_on ? chain_nb() : 0);
          if (!e && L.head && plan.pp.args.head_mt != g.head_mt) e = "conv_pp: head tiling mismatch";
        } else {
          e = plan_conv(&plan.tc, G, c->Pc, L.cin, L.cout, L.lin, L.lout, L.stride, L.pad, in_buf,
                        out_buf, out_q, g.wpack[li - 1], g.bias[li - 1], res,
                        conv1 ? 0 : L.res_mode, L.res_c, res_len, res_q, L.head ? g.fc_w : nullptr, head_base,
                        lane_sms, static_cast<size_t>(c->P_pad) * g.head_mt);
          if (!e && L.head && plan.tc.args.n_ntiles * plan.tc.args.mt_per_p != g.head_mt) e = "head tiling mismatch";
        }
        if (e) return fail(c, HB_E_INVALID, e);
        c->plans.push_back(plan);
        if (!conv1) cur = dst;
      }
    }
  }
  if (c->chain_on) {  // the chain's layer list: groups in order, layer-major; dependencies inside a group
    // HB_CHAIN_STEM_FLAGS=1: the stems publish tile counters (the stem_pp kernel serves every
    // chain-eligible width) and the chain's first layers start on published stem tiles
    const char* sf = getenv("HB_CHAIN_STEM_FLAGS");
    const char* hs = getenv("HB_STEM");
    // default off: the stem and the first layers share one HBM-bound phase, so overlapping them
    // measured no gain (tools/abtick.py: 0.626 ms whole-launch wait vs 0.639-0.709 ms with counters,
    // stem grids of 32-148 CTAs)
    bool flag_stems = (sf ? atoi(sf) : 0) != 0 && (hs ? atoi(hs) : 1) != 0 && c->n_chunks == 1;
    std::vector<ChainStemIn> stems;
    for (const Group& g : c->groups) {
      const LayerSpec& s0 = g.layers[0];
      const int oq = layer_in_q(g.layers[1], g.kind[1]);
      const int tpr = stem_tiles_per_row(c->W, oq, s0.cout);
      const int blocks = (act_rows_q(c->W, oq) + 1023) / 1024;  // 1024-position blocks per row
      flag_stems = flag_stems && tpr > 0;
      stems.push_back({tpr, tpr / blocks, act_rows_q(c->W, oq), c->Pc * static_cast<int>(g.mi.size())});
    }
    c->stem_sms = flag_stems ? (getenv("HB_STEM_SMS") ? atoi(getenv("HB_STEM_SMS")) : 0) : 0;
    int grid = c->num_sms;  // HB_CHAIN_SMS caps the persistent grid (tests: many items per CTA, stealing)
    if (const char* cs = getenv("HB_CHAIN_SMS")) grid = std::max(1, std::min(grid, atoi(cs)));
    c->chain_rest.assign(c->n_chunks - 1, ChainPlan());
    for (int ch = 0; ch < c->n_chunks; ++ch) {  // one chain plan per bed chunk (its head partials' rows)
      std::vector<ChainLayerIn> cl;
      double flops = 0, bytes = 0;
      for (size_t gi = 0; gi < c->groups.size(); ++gi) {
        const Group& g = c->groups[gi];
        const int first = static_cast<int>(cl.size());
        const double rows = static_cast<double>(c->Pc) * g.mi.size();
        for (size_t li = 1; li < g.layers.size(); ++li) {
          const LayerSpec& L = g.layers[li];
          ChainLayerIn x;
          x.plan = &c->plans[g.plan0[ch] + li - 1].pp;
          x.dep_in = li >= 2 ? first + static_cast<int>(li) - 2 : (flag_stems ? kChainDepStem : -1);
          x.dep_res = (li % 2 == 0 && li >= 3) ? first + static_cast<int>(li) - 3
                                               : (li == 2 && flag_stems ? kChainDepStem : -1);
          x.chain = static_cast<int>(gi);
          cl.push_back(x);
          flops += rows * 2.0 * L.cin * L.cout * kTaps * L.lout;
          bytes += rows * 2.0 * (static_cast<double>(L.cin) * L.lin + (L.head ? 0.0 : static_cast<double>(L.cout) * L.lout) +
                                 (L.res_mode ? static_cast<double>(L.res_c) * L.lin : 0.0));
        }
      }
      ChainPlan& cp = ch == 0 ? c->chain : c->chain_rest[ch - 1];
      const char* e = plan_chain(&cp, cl.data(), static_cast<int>(cl.size()), grid, flag_stems ? stems.data() : nullptr);
      if (e) return fail(c, HB_E_INVALID, e);
      cp.flops = flops;
      cp.bytes = bytes;
    }
  }
  CK(c, cudaMalloc(&c->d_heads, sizeof(HeadMember) * heads.size()));
  CK(c, cudaMemcpy(c->d_heads, heads.data(), sizeof(HeadMember) * heads.size(), cudaMemcpyHostToDevice));
  for (int ch = 0; c->chain_on && ch < c->n_chunks; ++ch) {
    // ensemble aggregation fused into each chunk's chain launch (HB_CHAIN_AGG=0: K5 after the last)
    ChainPlan& cp = ch == 0 ? c->chain : c->chain_rest[ch - 1];
    ChainArgs& ca = *cp.args;
    const char* ag = getenv("HB_CHAIN_AGG");
    ca.agg = (ag ? atoi(ag) : 1) != 0 ? 1 : 0;
    if (ca.agg) {
      unsigned target = 0;  // head-tile halves per bed: every member's last conv, per column tile
      for (int i = 0; i < cp.n_layers; ++i)
        if (ca.L[i].fc_w != nullptr) target += static_cast<unsigned>(ca.L[i].G * ca.L[i].nt_per_p * kEpiPartsChain);
      ca.n_heads = M;
      ca.P = c->P;
      ca.bed0 = ch * c->Pc;
      ca.n_beds = std::max(0, std::min(c->Pc, c->P - ch * c->Pc));  // (the last chunk's padding beds: none)
      ca.heads = c->d_heads;
      ca.member_logits = c->member_logits;
      ca.ens_prob = c->ens_prob;
      ca.ens_logit = c->ens_logit;
      ca.ens_sums = c->ens_sums;
      ca.wpos = ch + 1 == c->n_chunks ? c->wpos : nullptr;  // the tick's cursor: once, by the last chunk
      ca.advance = c->hop;
      ca.bed_target = target;
      if (!cp.d_bed) {
        CK(c, cudaMalloc(&cp.d_bed, sizeof(unsigned) * c->Pc));
        CK(c, cudaMemset(cp.d_bed, 0, sizeof(unsigned) * c->Pc));
      }
      ca.bed_ctr = cp.d_bed;
    }
  }
  // capture the tick into a graph
  cudaStream_t cap;
  CK(c, cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t g;
  CK(c, cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  const int rc = enqueue_tick(c, cap);
  cudaError_t ec = cudaStreamEndCapture(cap, &g);
  if (rc != HB_OK) {
    cudaStreamDestroy(cap);
    return rc;
  }
  CK(c, ec);
  CK(c, cudaGraphInstantiate(&c->graph, g, 0));
  cudaGraphDestroy(g);
  for (int k = 0; k < 2; ++k) {  // the same tick reading staged_io[k] + one D2H of the outputs into h_out[k]
    cudaGraph_t gio;
    c->staged = c->staged_io[k];
    CK(c, cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    const int rc2 = enqueue_tick(c, cap);
    const cudaError_t e2 = rc2 == HB_OK ? cudaMemcpyAsync(c->h_out[k], c->member_logits, sizeof(float) * out_floats,
                                                           cudaMemcpyDeviceToHost, cap)
                                        : cudaSuccess;
    cudaError_t ec2 = cudaStreamEndCapture(cap, &gio);
    if (rc2 != HB_OK) {
      cudaStreamDestroy(cap);
      return rc2;
    }
    CK(c, e2);
    CK(c, ec2);
    CK(c, cudaGraphInstantiate(&c->graph_io[k], gio, 0));
    cudaGraphDestroy(gio);
  }
  c->staged = c->staged_io[0];
  cudaStreamDestroy(cap);
  c->dirty = false;
  return HB_OK;
}

}  // namespace

extern "C" {

int hb_version(void) { return 1; }

const char* hb_last_error(const hb_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int hb_create(int device, const hb_config* cfg, hb_ctx** out) {
  if (!cfg || !out) return fail(nullptr, HB_E_INVALID, "null argument");
  if (cfg->max_patients < 1) return fail(nullptr, HB_E_CONFIG, "patients must be >= 1");
  if (cfg->n_leads < 1) return fail(nullptr, HB_E_CONFIG, "n_leads must be >= 1");
  if (cfg->window_len < kTaps) return fail(nullptr, HB_E_CONFIG, "window_len too short");
  if (cfg->hop < 1 || cfg->hop > cfg->window_len) return fail(nullptr, HB_E_CONFIG, "hop must be in [1, window_len]");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, HB_E_CUDA, "no CUDA device (there is no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(nullptr, HB_E_INVALID, "device ordinal out of range");
  if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, HB_E_CUDA, "cudaSetDevice failed");
  if (init_kernels() != cudaSuccess) return fail(nullptr, HB_E_CUDA, "kernel attribute setup failed");
  hb_ctx* c = new hb_ctx();
  c->device = device;
  c->P = cfg->max_patients;
  c->leads = cfg->n_leads;
  c->fs = cfg->fs;
  c->W = cfg->window_len;
  c->hop = cfg->hop;
  c->R = cfg->ring_len > 0 ? cfg->ring_len : round_up(cfg->window_len + cfg->hop, 256);
  c->keep = cfg->keep_windows;
  if (getenv("HB_LANES")) c->max_lanes = std::max(1, atoi(getenv("HB_LANES")));
  if (getenv("HB_NO_GROUP")) c->group_off = atoi(getenv("HB_NO_GROUP"));
  if (getenv("HB_MAX_GROUP")) c->max_group = std::max(1, std::min(kMaxGroup, atoi(getenv("HB_MAX_GROUP"))));
  if (getenv("HB_ACT_BUDGET_GB")) c->act_budget = atof(getenv("HB_ACT_BUDGET_GB")) * 1e9;
  if (c->R < c->W) {
    delete c;
    return fail(nullptr, HB_E_CONFIG, "ring_len must be >= window_len");
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  const size_t S = static_cast<size_t>(c->P) * c->leads;
  bool ok = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMalloc(&c->ring, S * (c->R + c->W) * sizeof(float)) == cudaSuccess &&  // + mirror of W
            cudaMemset(c->ring, 0, S * (c->R + c->W) * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&c->staged_io[0], S * c->hop * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&c->staged_io[1], S * c->hop * sizeof(float)) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->h2d_done[0], cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->h2d_done[1], cudaEventDisableTiming) == cudaSuccess &&
            cudaMalloc(&c->prefill, S * c->R * sizeof(float)) == cudaSuccess &&
            cudaMalloc(&c->wpos, sizeof(long long)) == cudaSuccess &&
            cudaMemset(c->wpos, 0, sizeof(long long)) == cudaSuccess &&
            cudaMalloc(&c->stats, S * 2 * sizeof(float)) == cudaSuccess &&
            cudaEventCreate(&c->t0) == cudaSuccess && cudaEventCreate(&c->t1) == cudaSuccess;
  if (ok) c->staged = c->staged_io[0];
  if (ok && c->keep) ok = cudaMalloc(&c->raw, S * c->W * sizeof(float)) == cudaSuccess;
  if (!ok) {
    hb_destroy(c);
    return fail(nullptr, HB_E_CUDA, "device allocation failed");
  }
  *out = c;
  return HB_OK;
}

int hb_destroy(hb_ctx* c) {
  if (!c) return HB_OK;
  cudaSetDevice(c->device);
  if (c->own) cudaStreamSynchronize(c->own);
  free_selection(c);
  for (auto& kv : c->members) free_member(kv.second);
  cudaFree(c->ring);
  cudaFree(c->staged_io[0]);
  cudaFree(c->staged_io[1]);
  for (int k = 0; k < 2; ++k)
    if (c->h2d_done[k]) cudaEventDestroy(c->h2d_done[k]);
  if (c->copy) cudaStreamDestroy(c->copy);
  cudaFree(c->prefill);
  cudaFree(c->wpos);
  cudaFree(c->xn);
  cudaFree(c->raw);
  cudaFree(c->stats);
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  for (int k = 0; k < 2; ++k)
    if (c->io_done[k]) cudaEventDestroy(c->io_done[k]);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
  return HB_OK;
}

int hb_add_member(hb_ctx* c, int idx, int lead, int width, int depth, const float* params, size_t n_floats) {
  if (!c || !params) return fail(c, HB_E_INVALID, "null argument");
  if (idx < 0) return fail(c, HB_E_INVALID, "member idx must be >= 0");
  if (lead < 0 || lead >= c->leads)
    return fail(c, HB_E_CONFIG, "rates: no stream configured for lead " + std::to_string(lead));
  if (width < 8 || width % 8 || width > 128 || depth < 1) return fail(c, HB_E_INVALID, "unsupported width/depth");
  if (c->io_busy[0] || c->io_busy[1])
    return fail(c, HB_E_STATE, "a submitted tick is uncollected; collect it before registering members");
  cudaSetDevice(c->device);
  Member m;
  m.idx = idx;
  m.lead = lead;
  m.width = width;
  m.depth = depth;
  m.layers = member_layers(width, depth, c->W);
  size_t need = 0;
  for (auto& L : m.layers) need += static_cast<size_t>(L.cout) * L.cin * kTaps + L.cout;
  const int c_last = m.layers.back().cout;
  need += c_last + 1;
  if (n_floats != need)
    return fail(c, HB_E_INVALID, "params blob has " + std::to_string(n_floats) + " floats, expected " +
                                     std::to_string(need));
  const float* p = params;
  const LayerSpec& s0 = m.layers[0];
  CK(c, cudaMalloc(&m.stem_w, sizeof(float) * s0.cout * kTaps));
  CK(c, cudaMemcpy(m.stem_w, p, sizeof(float) * s0.cout * kTaps, cudaMemcpyHostToDevice));
  p += s0.cout * kTaps;
  CK(c, cudaMalloc(&m.stem_b, sizeof(float) * s0.cout));
  CK(c, cudaMemcpy(m.stem_b, p, sizeof(float) * s0.cout, cudaMemcpyHostToDevice));
  p += s0.cout;
  for (size_t li = 1; li < m.layers.size(); ++li) {
    const LayerSpec& L = m.layers[li];
    // both weight images: the kernel per layer is chosen when the selection is built
    for (int kind = KIND_TC; kind <= KIND_PP; ++kind) {
      if (kind == KIND_PP && !pp_eligible(L)) {
        m.wpp.push_back(nullptr);
        continue;
      }
      const size_t wb = layer_wbytes(L, kind);
      std::vector<uint16_t> img(wb / 2);
      layer_pack(L, kind, p, img.data());
      uint8_t* dw;
      CK(c, cudaMalloc(&dw, wb));
      CK(c, cudaMemcpy(dw, img.data(), wb, cudaMemcpyHostToDevice));
      (kind == KIND_PP ? m.wpp : m.wpack).push_back(dw);
    }
    p += static_cast<size_t>(L.cout) * L.cin * kTaps;
    const int bn = conv_bn(L.cout);
    const int nbias = ((round_up(L.cout, 16) + bn - 1) / bn) * bn;
    std::vector<float> bias(nbias, 0.f);
    std::copy(p, p + L.cout, bias.begin());
    float* db;
    CK(c, cudaMalloc(&db, sizeof(float) * nbias));
    CK(c, cudaMemcpy(db, bias.data(), sizeof(float) * nbias, cudaMemcpyHostToDevice));
    m.bias.push_back(db);
    p += L.cout;
  }
  CK(c, cudaMalloc(&m.fc_w, sizeof(float) * c_last));
  CK(c, cudaMemcpy(m.fc_w, p, sizeof(float) * c_last, cudaMemcpyHostToDevice));
  p += c_last;
  m.fc_b = *p;
  m.head_mt = (m.layers.back().lout + kBM - 1) / kBM;
  for (auto& L : m.layers) {
    m.flops += 2.0 * L.cin * L.cout * kTaps * L.lout;
    m.bytes += 2.0 * (static_cast<double>(L.cin) * L.lin + (L.head ? 0.0 : static_cast<double>(L.cout) * L.lout));
  }
  auto it = c->members.find(idx);
  if (it != c->members.end()) free_member(it->second);
  c->members[idx] = m;
  c->dirty = true;
  return HB_OK;
}

int hb_set_selector(hb_ctx* c, const uint8_t* bits, int n) {
  if (!c || !bits) return fail(c, HB_E_INVALID, "null argument");
  std::vector<int> sel;
  for (int k = 0; k < n; ++k) {
    if (bits[k] > 1) return fail(c, HB_E_INVALID, "selector bits must be 0 or 1");
    if (bits[k]) {
      if (!c->members.count(k)) return fail(c, HB_E_STATE, "selected member " + std::to_string(k) + " not registered");
      sel.push_back(k);
    }
  }
  if (sel.empty()) return fail(c, HB_E_EMPTY, "cannot serve an empty ensemble");
  if (static_cast<int>(sel.size()) > kMaxMembers) return fail(c, HB_E_INVALID, "too many selected members");
  if (sel != c->selected && (c->io_busy[0] || c->io_busy[1]))
    return fail(c, HB_E_STATE, "a submitted tick is uncollected; collect it before changing the selector");
  if (sel != c->selected) {
    c->selected = sel;
    c->dirty = true;
  }
  return HB_OK;
}

int hb_selected(const hb_ctx* c, int* idx_out, int cap) {
  if (!c) return -1;
  const int M = static_cast<int>(c->selected.size());
  for (int i = 0; i < M && i < cap && idx_out; ++i) idx_out[i] = c->selected[i];
  return M;
}

int hb_ingest(hb_ctx* c, const float* samples, int n, void* stream) {
  if (!c || (!samples && n > 0)) return fail(c, HB_E_INVALID, "null argument");
  NvtxRange nv("hb:ingest");
  if (n < 0) return fail(c, HB_E_INVALID, "n_per_stream must be >= 0");
  cudaSetDevice(c->device);
  cudaStream_t st = pick(c, stream);
  const size_t S = static_cast<size_t>(c->P) * c->leads;
  for (int done = 0; done < n;) {
    const int chunk = std::min(n - done, c->R);
    // gather columns [done, done+chunk) of every stream into the contiguous prefill buffer
    CK(c, cudaMemcpy2DAsync(c->prefill, sizeof(float) * chunk, samples + done, sizeof(float) * n,
                            sizeof(float) * chunk, S, cudaMemcpyHostToDevice, st));
    CK(c, launch_ingest_window(c->prefill, c->ring, c->wpos, c->P, c->leads, chunk, c->R, c->W, nullptr, 0, nullptr,
                               nullptr, st));
    CK(c, launch_advance(c->wpos, chunk, st));
    done += chunk;
  }
  CK(c, cudaStreamSynchronize(st));
  return HB_OK;
}

int hb_stage_device(hb_ctx* c, const float* dev, void* stream) {
  if (!c || !dev) return fail(c, HB_E_INVALID, "null argument");
  cudaSetDevice(c->device);
  CK(c, cudaMemcpyAsync(c->staged, dev, sizeof(float) * c->P * c->leads * c->hop, cudaMemcpyDeviceToDevice,
                        pick(c, stream)));
  return HB_OK;
}

int hb_tick_device(hb_ctx* c, void* stream) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  cudaSetDevice(c->device);
  const int rc = build_selection(c);
  if (rc) return rc;
  cudaStream_t st = pick(c, stream);
  CK(c, cudaEventRecord(c->t0, st));
  CK(c, cudaGraphLaunch(c->graph, st));
  CK(c, cudaEventRecord(c->t1, st));
  c->timed = true;
  return HB_OK;
}

namespace {
// overlap_h2d: the H2D runs on the copy stream into the slot's staging buffer
// (pipelined submit); otherwise in-stream (blocking tick: lowest latency).
int tick_submit(hb_ctx* c, const float* samples, int slot, void* stream, bool overlap_h2d);
}  // namespace

int hb_tick_submit(hb_ctx* c, const float* samples, int slot, void* stream) {
  return tick_submit(c, samples, slot, stream, true);
}

namespace {
int tick_submit(hb_ctx* c, const float* samples, int slot, void* stream, bool overlap_h2d) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  NvtxRange nv("hb:tick_submit");
  if (slot < 0 || slot > 1) return fail(c, HB_E_INVALID, "slot must be 0 or 1");
  cudaSetDevice(c->device);
  cudaStream_t st = pick(c, stream);
  // the busy check comes first: rebuilding a selection frees both slots' pinned outputs
  if (c->io_busy[slot]) return fail(c, HB_E_STATE, "slot " + std::to_string(slot) + " has an uncollected tick");
  if (c->dirty && (c->io_busy[0] || c->io_busy[1]))
    return fail(c, HB_E_STATE, "the selection changed while a submitted tick is uncollected; collect it first");
  const int rc = build_selection(c);
  if (rc) return rc;
  if (samples && overlap_h2d) {  // H2D on the copy stream into this slot's staging buffer: overlaps the tick in flight
    CK(c, cudaMemcpyAsync(c->staged_io[slot], samples, sizeof(float) * c->P * c->leads * c->hop,
                          cudaMemcpyHostToDevice, c->copy));
    CK(c, cudaEventRecord(c->h2d_done[slot], c->copy));
    CK(c, cudaStreamWaitEvent(st, c->h2d_done[slot], 0));
  } else if (samples) {
    CK(c, cudaMemcpyAsync(c->staged_io[slot], samples, sizeof(float) * c->P * c->leads * c->hop,
                          cudaMemcpyHostToDevice, st));
  } else if (slot != 0) {
    return fail(c, HB_E_INVALID, "samples staged with hb_stage_device are in slot 0");
  }
  CK(c, cudaEventRecord(c->t0, st));
  CK(c, cudaGraphLaunch(c->graph_io[slot], st));
  CK(c, cudaEventRecord(c->t1, st));
  if (!c->io_done[slot]) CK(c, cudaEventCreateWithFlags(&c->io_done[slot], cudaEventDisableTiming));
  CK(c, cudaEventRecord(c->io_done[slot], st));
  c->timed = true;
  c->io_busy[slot] = true;
  c->slot_M[slot] = static_cast<int>(c->selected.size());
  return HB_OK;
}

}  // namespace

int hb_tick_collect(hb_ctx* c, int slot, float* member_logits, float* ens_prob, float* ens_mean_logit) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  NvtxRange nv("hb:tick_collect");
  if (slot < 0 || slot > 1) return fail(c, HB_E_INVALID, "slot must be 0 or 1");
  if (!c->io_busy[slot]) return fail(c, HB_E_STATE, "slot " + std::to_string(slot) + " has no submitted tick");
  cudaSetDevice(c->device);
  c->io_busy[slot] = false;
  CK(c, cudaEventSynchronize(c->io_done[slot]));
  // the layout of the tick submitted into this slot, not of the selection now
  const size_t P = c->P, M = static_cast<size_t>(c->slot_M[slot]);
  const float* h = c->h_out[slot];
  if (member_logits) std::memcpy(member_logits, h, sizeof(float) * P * M);
  if (ens_prob) std::memcpy(ens_prob, h + P * M, sizeof(float) * P);
  if (ens_mean_logit) std::memcpy(ens_mean_logit, h + P * M + P, sizeof(float) * P);
  return HB_OK;
}

int hb_tick(hb_ctx* c, const float* samples, float* member_logits, float* ens_prob, float* ens_mean_logit,
            void* stream) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  NvtxRange nv("hb:tick");
  const bool host_out = member_logits || ens_prob || ens_mean_logit;
  if (host_out) {
    int slot = c->io_busy[0] ? (c->io_busy[1] ? -1 : 1) : 0;
    if (slot < 0) return fail(c, HB_E_STATE, "both tick slots hold uncollected ticks");
    const int rc = tick_submit(c, samples, slot, stream, false);
    return rc ? rc : hb_tick_collect(c, slot, member_logits, ens_prob, ens_mean_logit);
  }
  cudaSetDevice(c->device);
  cudaStream_t st = pick(c, stream);
  const int rc = build_selection(c);
  if (rc) return rc;
  if (samples)
    CK(c, cudaMemcpyAsync(c->staged, samples, sizeof(float) * c->P * c->leads * c->hop, cudaMemcpyHostToDevice, st));
  CK(c, cudaEventRecord(c->t0, st));
  CK(c, cudaGraphLaunch(c->graph, st));
  CK(c, cudaEventRecord(c->t1, st));
  c->timed = true;
  return HB_OK;
}

int hb_profile_tick(hb_ctx* c, void* stream, int cap, int* kinds, float* ms, double* flops, double* bytes) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  cudaSetDevice(c->device);
  const int rc0 = build_selection(c);
  if (rc0) return rc0;
  cudaStream_t st = pick(c, stream);
  std::vector<cudaEvent_t> ev;
  cudaEvent_t start;
  CK(c, cudaEventCreate(&start));
  CK(c, cudaEventRecord(start, st));
  ProfRec pr;
  pr.ev = &ev;
  const int rc = enqueue_tick(c, st, &pr);
  CK(c, cudaStreamSynchronize(st));
  const int n = static_cast<int>(ev.size());
  cudaEvent_t prev = start;
  for (int i = 0; i < n; ++i) {
    float t = 0.f;
    cudaEventElapsedTime(&t, prev, ev[i]);
    if (i < cap) {
      if (kinds) kinds[i] = pr.kind[i];
      if (ms) ms[i] = t;
      if (flops) flops[i] = pr.flops[i];
      if (bytes) bytes[i] = pr.bytes[i];
    }
    prev = ev[i];
  }
  for (auto e : ev) cudaEventDestroy(e);
  cudaEventDestroy(start);
  if (rc) return rc;
  return n;
}

int hb_last_tick_ms(hb_ctx* c, float* ms) {
  if (!c || !ms) return fail(c, HB_E_INVALID, "null argument");
  if (!c->timed) return fail(c, HB_E_STATE, "no tick has run yet");
  cudaSetDevice(c->device);
  CK(c, cudaEventSynchronize(c->t1));
  CK(c, cudaEventElapsedTime(ms, c->t0, c->t1));
  return HB_OK;
}

int hb_time_tick(hb_ctx* c, int reps, float* median_ms) {
  if (!c || !median_ms || reps < 1) return fail(c, HB_E_INVALID, "bad argument");
  cudaSetDevice(c->device);
  const int rc = build_selection(c);
  if (rc) return rc;
  cudaStream_t st = c->own;
  // warm-up launch, then `reps` individually bracketed launches; the stream
  // cursor advances like a real tick (the data is whatever the rings hold)
  CK(c, cudaGraphLaunch(c->graph, st));
  std::vector<float> t(reps);
  for (int i = 0; i < reps; ++i) {
    CK(c, cudaEventRecord(c->t0, st));
    CK(c, cudaGraphLaunch(c->graph, st));
    CK(c, cudaEventRecord(c->t1, st));
    CK(c, cudaEventSynchronize(c->t1));
    CK(c, cudaEventElapsedTime(&t[i], c->t0, c->t1));
  }
  std::sort(t.begin(), t.end());
  *median_ms = t[reps / 2];
  return HB_OK;
}

int hb_prepare(hb_ctx* c) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  cudaSetDevice(c->device);
  if (c->dirty && (c->io_busy[0] || c->io_busy[1]))
    return fail(c, HB_E_STATE, "the selection changed while a submitted tick is uncollected; collect it first");
  const int rc = build_selection(c);
  if (rc) return rc;
  CK(c, cudaGraphUpload(c->graph, c->own));
  for (int k = 0; k < 2; ++k) CK(c, cudaGraphUpload(c->graph_io[k], c->own));
  CK(c, cudaStreamSynchronize(c->own));
  return HB_OK;
}

int hb_chain_profile(hb_ctx* c, unsigned long long* out, int cap) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  if (!c->chain_on || !c->chain.d_prof) return 0;
  cudaSetDevice(c->device);
  CK(c, cudaDeviceSynchronize());
  const int n = std::min(cap, c->chain.grid);
  if (out && n > 0) CK(c, cudaMemcpy(out, c->chain.d_prof, sizeof(unsigned long long) * 16 * n, cudaMemcpyDeviceToHost));
  return c->chain.grid;
}

int hb_chain_trace(hb_ctx* c, unsigned long long* trace, int* items, int cap) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  if (!c->chain_on || !c->chain.d_trace) return 0;
  cudaSetDevice(c->device);
  CK(c, cudaDeviceSynchronize());
  const int n = std::min(cap, c->chain.n_items);
  if (trace && n > 0)
    CK(c, cudaMemcpy(trace, c->chain.d_trace, sizeof(unsigned long long) * 5 * n, cudaMemcpyDeviceToHost));
  if (items && n > 0) CK(c, cudaMemcpy(items, c->chain.d_items, sizeof(int) * n, cudaMemcpyDeviceToHost));
  return c->chain.n_items;
}

int hb_device_outputs(const hb_ctx* c, float** ml, float** ep, float** el) {
  if (!c || !c->member_logits) return HB_E_STATE;
  if (ml) *ml = c->member_logits;
  if (ep) *ep = c->ens_prob;
  if (el) *el = c->ens_logit;
  return HB_OK;
}

int hb_device_sums(const hb_ctx* c, float** sums) {
  if (!c || !c->ens_sums || !sums) return HB_E_STATE;
  *sums = c->ens_sums;
  return HB_OK;
}

int hb_finalize_sums(const float* sums, int P, int m_total, float* prob, float* logit, void* stream) {
  if (!sums || !prob || !logit || P < 1 || m_total < 1) return fail(nullptr, HB_E_INVALID, "bad argument");
  const cudaError_t e = launch_finalize(sums, P, m_total, prob, logit, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(nullptr, HB_E_CUDA, cudaGetErrorString(e));
  return HB_OK;
}

int hb_last_windows(hb_ctx* c, float* raw, float* stats, void* stream) {
  if (!c) return fail(c, HB_E_INVALID, "null argument");
  cudaSetDevice(c->device);
  cudaStream_t st = pick(c, stream);
  const size_t S = static_cast<size_t>(c->P) * c->leads;
  if (raw) {
    if (!c->keep) return fail(c, HB_E_STATE, "context created without keep_windows");
    CK(c, cudaMemcpyAsync(raw, c->raw, sizeof(float) * S * c->W, cudaMemcpyDeviceToHost, st));
  }
  if (stats) CK(c, cudaMemcpyAsync(stats, c->stats, sizeof(float) * S * 2, cudaMemcpyDeviceToHost, st));
  CK(c, cudaStreamSynchronize(st));
  return HB_OK;
}

int hb_tick_work(const hb_ctx* c, double* flops, double* bytes) {
  if (!c) return HB_E_INVALID;
  double f = 0, b = 0;
  for (int idx : c->selected) {
    const Member& m = c->members.at(idx);
    f += m.flops;
    b += m.bytes;
  }
  if (flops) *flops = f * c->P;
  if (bytes) *bytes = b * c->P;
  return HB_OK;
}

int hb_last_normalized(hb_ctx* c, uint16_t* xn, void* stream) {
  if (!c || !xn) return fail(c, HB_E_INVALID, "null argument");
  if (!c->xn) return fail(c, HB_E_STATE, "no selection built yet (tick first)");
  cudaSetDevice(c->device);
  cudaStream_t st = pick(c, stream);
  // device layout [leads][P_pad][roundup(W, 8)] -> host [leads][P][W]
  const size_t Wp = round_up(c->W, 8);
  for (int lead = 0; lead < c->leads; ++lead)
    CK(c, cudaMemcpy2DAsync(xn + static_cast<size_t>(lead) * c->P * c->W, sizeof(uint16_t) * c->W,
                            c->xn + static_cast<size_t>(lead) * c->P_pad * Wp, sizeof(uint16_t) * Wp,
                            sizeof(uint16_t) * c->W, c->P, cudaMemcpyDeviceToHost, st));
  CK(c, cudaStreamSynchronize(st));
  return HB_OK;
}

int hb_member_layers(int width, int depth, int window, int* out, int cap) {
  if (width < 8 || width % 8 || depth < 1 || window < kTaps || cap < 0) return -HB_E_INVALID;
  const std::vector<LayerSpec> v = member_layers(width, depth, window);
  for (int i = 0; i < static_cast<int>(v.size()) && i < cap && out; ++i) {
    const LayerSpec& L = v[i];
    const int row[9] = {L.cin, L.cout, L.stride, L.lin, L.lout, L.pad, L.res_mode, L.res_c, L.head};
    std::copy(row, row + 9, out + 9 * i);
  }
  return static_cast<int>(v.size());
}

// ----------------------------------------------------------------- test entry points

int hb_op_conv1d_q(const void* in, int P, int cin, int lin, int stride, const float* w_host, const float* b_host,
                   int cout, const void* res, int res_mode, int res_c, int res_len, int res_q, void* out, int out_q,
                   const float* fc_w_host, float* head_out, int kind, void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (init_kernels() != cudaSuccess) return fail(nullptr, HB_E_CUDA, "kernel attribute setup failed");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int lout = (lin + stride - 1) / stride;
  const int tot = (lout - 1) * stride + kTaps - lin;
  const int pad = tot > 0 ? tot / 2 : 0;
  if (kind < 0) kind = layer_kind({cin, cout, stride, lin, lout, pad, res_mode, res_c, fc_w_host ? 1 : 0});
  const LayerSpec spec{cin, cout, stride, lin, lout, pad, res_mode, res_c, fc_w_host ? 1 : 0};
  const size_t wb = layer_wbytes(spec, kind);
  std::vector<uint16_t> img(wb / 2);
  layer_pack(spec, kind, w_host, img.data());
  const int nbias = static_cast<int>(bias_len(cout));
  std::vector<float> bias(nbias, 0.f);
  std::copy(b_host, b_host + cout, bias.begin());
  uint8_t* dw = nullptr;
  float *db = nullptr, *dfc = nullptr;
  hb_ctx* none = nullptr;
  CK(none, cudaMalloc(&dw, wb));
  CK(none, cudaMemcpy(dw, img.data(), wb, cudaMemcpyHostToDevice));
  CK(none, cudaMalloc(&db, sizeof(float) * nbias));
  CK(none, cudaMemcpy(db, bias.data(), sizeof(float) * nbias, cudaMemcpyHostToDevice));
  if (fc_w_host) {
    CK(none, cudaMalloc(&dfc, sizeof(float) * cout));
    CK(none, cudaMemcpy(dfc, fc_w_host, sizeof(float) * cout, cudaMemcpyHostToDevice));
  }
  LayerPlan plan;
  plan.kind = kind;
  const char* e;
  if (kind == KIND_PP)
    e = plan_pp(&plan.pp, 1, P, cin, cout, lin, lout, stride, pad, static_cast<const __half*>(in),
                static_cast<__half*>(out), out_q, dw, db, static_cast<const __half*>(res), res_mode, res_c,
                res_len > 0 ? res_len : lout, res_q, sms, layer_zc(spec), dfc, head_out, 0);
  else
    e = plan_conv(&plan.tc, 1, P, cin, cout, lin, lout, stride, pad, static_cast<const __half*>(in),
                  static_cast<__half*>(out), out_q, dw, db, static_cast<const __half*>(res), res_mode, res_c,
                  res_len > 0 ? res_len : lout, res_q, dfc, head_out, sms);
  int rc = HB_OK;
  if (e) {
    g_create_err = e;
    rc = HB_E_INVALID;
  } else {
    cudaError_t ce = launch_layer(plan, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) {
      g_create_err = std::string("conv launch: ") + cudaGetErrorString(ce);
      rc = HB_E_CUDA;
    }
  }
  cudaFree(dw);
  cudaFree(db);
  cudaFree(dfc);
  return rc;
}

int hb_op_conv1d(const void* in, int P, int cin, int lin, int stride, const float* w_host, const float* b_host,
                 int cout, const void* res, int res_mode, int res_c, int res_len, void* out, int out_split,
                 const float* fc_w_host, float* head_out, void* stream) {
  return hb_op_conv1d_q(in, P, cin, lin, stride, w_host, b_host, cout, res, res_mode, res_c, res_len,
                        res_mode == 2 ? 2 : 1, out, out_split ? 2 : 1, fc_w_host, head_out, KIND_TC, stream);
}

int hb_conv_head_mt(int P, int cin, int cout, int lin, int stride, int res_mode, int kind) {
  const int lout = (lin + stride - 1) / stride;
  const int tot = (lout - 1) * stride + kTaps - lin;
  const LayerSpec L{cin, cout, stride, lin, lout, tot > 0 ? tot / 2 : 0, res_mode, cin < cout ? cin : cout, 1};
  if (kind < 0) kind = layer_kind(L);
  if (kind == KIND_PP) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return pp_head_mt(L, 1, P, sms);
  }
  return hb_conv_mt(cin, cout, lin, stride, 1);
}

int hb_conv_kind(int cin, int cout, int stride, int head) {
  return layer_kind({cin, cout, stride, 0, 0, 0, 0, 0, head});
}

int hb_conv_mt(int cin, int cout, int lin, int stride, int head) {
  const int lout = (lin + stride - 1) / stride;
  const int rows = head ? lout : act_rows(lout, 0);
  const int sm = conv_stride_m(conv_fold(cin, cout, stride));
  const int bn = conv_bn(cout), nnt = (round_up(cout, 16) + bn - 1) / bn;
  return (head ? nnt : 1) * ((rows + sm - 1) / sm);
}

int hb_bench_conv_k(int P, int cin, int cout, int lin, int stride, int res_mode, int kind, int iters, float* ms_out) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (init_kernels() != cudaSuccess) return fail(nullptr, HB_E_CUDA, "kernel attribute setup failed");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int lout = (lin + stride - 1) / stride;
  const int tot = (lout - 1) * stride + kTaps - lin;
  const int pad = tot > 0 ? tot / 2 : 0;
  const size_t in_b = static_cast<size_t>(P) * cin * plane_rows_max(lin) * 2;
  const size_t out_b = static_cast<size_t>(P) * cout * plane_rows_max(lout) * 2;
  if (kind < 0) kind = layer_kind({cin, cout, stride, lin, lout, pad, res_mode, cin < cout ? cin : cout, 0});
  const LayerSpec spec{cin, cout, stride, lin, lout, pad, res_mode, cin < cout ? cin : cout, 0};
  const size_t wb = layer_wbytes(spec, kind);
  const int bn = conv_bn(cout);
  const int nbias = ((round_up(cout, 16) + bn - 1) / bn) * bn;
  void *din = nullptr, *dout = nullptr, *dres = nullptr, *dw = nullptr, *db = nullptr;
  hb_ctx* none = nullptr;
  CK(none, cudaMalloc(&din, in_b));
  CK(none, cudaMemset(din, 0, in_b));
  CK(none, cudaMalloc(&dout, out_b));
  // the shortcut tensor: x at the output length (identity) or twice the input length (maxpool)
  const size_t res_b = std::max({in_b, out_b, static_cast<size_t>(P) * std::min(cin, cout) * plane_rows_max(2 * lin) * 2});
  CK(none, cudaMalloc(&dres, res_b));
  CK(none, cudaMemset(dres, 0, res_b));
  CK(none, cudaMalloc(&dw, wb));
  CK(none, cudaMemset(dw, 0, wb));
  CK(none, cudaMalloc(&db, nbias * 4));
  CK(none, cudaMemset(db, 0, nbias * 4));
  LayerPlan plan;
  plan.kind = kind;
  const int in_q = layer_in_q(spec, kind);
  const int out_q = kind == KIND_PP ? pp_phases(cout) : 1;  // as if feeding a like layer
  const int res_q = res_mode == 2 ? in_q : out_q;
  const char* e;
  if (kind == KIND_PP)
    e = plan_pp(&plan.pp, 1, P, cin, cout, lin, lout, stride, pad, static_cast<const __half*>(din),
                static_cast<__half*>(dout), out_q, static_cast<uint8_t*>(dw), static_cast<float*>(db),
                res_mode ? static_cast<const __half*>(dres) : nullptr, res_mode, cin < cout ? cin : cout,
                res_mode == 2 ? 2 * lin : lout, res_q, sms, layer_zc(spec));
  else
    e = plan_conv(&plan.tc, 1, P, cin, cout, lin, lout, stride, pad, static_cast<const __half*>(din),
                  static_cast<__half*>(dout), out_q, static_cast<uint8_t*>(dw), static_cast<float*>(db),
                  res_mode ? static_cast<const __half*>(dres) : nullptr, res_mode, cin < cout ? cin : cout,
                  res_mode == 2 ? 2 * lin : lout, res_q, nullptr, nullptr, sms);
  int rc = HB_OK;
  unsigned long long* dprof = nullptr;
  if (!e && kind == KIND_PP && (plan.pp.args.dbg & 16)) {
    cudaMalloc(&dprof, sizeof(unsigned long long) * 8 * plan.pp.grid);
    cudaMemset(dprof, 0, sizeof(unsigned long long) * 8 * plan.pp.grid);
    plan.pp.args.prof = dprof;
  }
  if (!e && kind == KIND_TC && (plan.tc.args.dbg & 8)) {
    cudaMalloc(&dprof, sizeof(unsigned long long) * 8 * plan.tc.grid);
    cudaMemset(dprof, 0, sizeof(unsigned long long) * 8 * plan.tc.grid);
    plan.tc.args.prof = dprof;
  }
  if (e) {
    g_create_err = e;
    rc = HB_E_INVALID;
  } else {
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) launch_layer(plan, st);
    cudaEventRecord(a, st);
    for (int i = 0; i < iters; ++i) launch_layer(plan, st);
    cudaEventRecord(b, st);
    cudaError_t ce = cudaStreamSynchronize(st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(st);
    if (dprof && kind == KIND_PP) {
      const int grid = plan.pp.grid;
      std::vector<unsigned long long> h(8 * grid);
      cudaMemcpy(h.data(), dprof, h.size() * 8, cudaMemcpyDeviceToHost);
      double sum[8] = {0};
      for (int i = 0; i < grid; ++i)
        for (int k = 0; k < 8; ++k) sum[k] += static_cast<double>(h[i * 8 + k]) / grid;
      const double tiles = static_cast<double>(plan.pp.args.num_tiles) / grid;
      fprintf(stderr, "[pp prof] nb=%d stages=%d tiles/CTA %.1f | per tile (cycles): mma wait_acc %.0f wait_b %.0f total %.0f | epi(wg0) wait %.0f work %.0f (per its tile, %.1f tiles)\n",
              plan.pp.args.nb, plan.pp.args.n_stages, tiles, sum[0] / tiles, sum[1] / tiles, sum[2] / tiles,
              sum[3] / sum[6], sum[4] / sum[6], sum[6]);
      cudaFree(dprof);
      dprof = nullptr;
    }
    if (dprof) {
      std::vector<unsigned long long> h(8 * plan.tc.grid);
      cudaMemcpy(h.data(), dprof, h.size() * 8, cudaMemcpyDeviceToHost);
      double sum[8] = {0};
      for (int i = 0; i < plan.tc.grid; ++i)
        for (int k = 0; k < 8; ++k) sum[k] += static_cast<double>(h[i * 8 + k]) / plan.tc.grid;
      const double tiles = static_cast<double>(plan.tc.args.num_tiles) / plan.tc.grid;
      fprintf(stderr, "[prof] per tile (cycles): mma wait_acc %.0f wait_a %.0f issue %.0f | epi wait %.0f work %.0f | epi total/tile %.0f (tiles/CTA %.1f)\n",
              sum[0] / tiles, sum[1] / tiles, sum[2] / tiles, sum[3] / tiles, sum[4] / tiles, sum[5] / tiles, tiles);
      cudaFree(dprof);
    }
    if (ce != cudaSuccess) {
      g_create_err = cudaGetErrorString(ce);
      rc = HB_E_CUDA;
    }
  }
  cudaFree(din);
  cudaFree(dout);
  cudaFree(dres);
  cudaFree(dw);
  cudaFree(db);
  return rc;
}

// Back-to-back stem launches (zero data) for timing experiments: G members of Pm rows.
int hb_bench_stem(int G, int Pm, int L, int cout, int out_q, int iters, float* ms_out) {
  if (init_kernels() != cudaSuccess) return fail(nullptr, HB_E_CUDA, "kernel attribute setup failed");
  if (G < 1 || G > kMaxGroup || Pm < 1 || L < 16 || iters < 1) return fail(nullptr, HB_E_INVALID, "bad stem bench shape");
  hb_ctx* none = nullptr;
  const int Lp = round_up(L, 8);
  void *x = nullptr, *w = nullptr, *b = nullptr, *out = nullptr;
  const size_t out_b = static_cast<size_t>(G) * Pm * cout * plane_rows_max(L) * 2;
  CK(none, cudaMalloc(&x, static_cast<size_t>(G) * Pm * Lp * 2));
  CK(none, cudaMemset(x, 0, static_cast<size_t>(G) * Pm * Lp * 2));
  CK(none, cudaMalloc(&w, sizeof(float) * cout * kTaps));
  CK(none, cudaMemset(w, 0, sizeof(float) * cout * kTaps));
  CK(none, cudaMalloc(&b, sizeof(float) * cout));
  CK(none, cudaMemset(b, 0, sizeof(float) * cout));
  CK(none, cudaMalloc(&out, out_b));
  std::vector<StemMember> m(G);
  for (int g = 0; g < G; ++g)
    m[g] = StemMember{static_cast<const __half*>(x) + static_cast<size_t>(g) * Pm * Lp, static_cast<float*>(w),
                      static_cast<float*>(b)};
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaError_t ce = cudaSuccess;
  for (int i = 0; i < 3 && ce == cudaSuccess; ++i)
    ce = launch_stem(m.data(), G, Lp, Pm, L, out_q, cout, (kTaps - 1) / 2, static_cast<__half*>(out), st);
  cudaEventRecord(e0, st);
  for (int i = 0; i < iters && ce == cudaSuccess; ++i)
    ce = launch_stem(m.data(), G, Lp, Pm, L, out_q, cout, (kTaps - 1) / 2, static_cast<__half*>(out), st);
  cudaEventRecord(e1, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaFree(x);
  cudaFree(w);
  cudaFree(b);
  cudaFree(out);
  if (ce != cudaSuccess) return fail(none, HB_E_CUDA, cudaGetErrorString(ce));
  return HB_OK;
}

int hb_bench_conv(int P, int cin, int cout, int lin, int stride, int res_mode, int iters, float* ms_out) {
  return hb_bench_conv_k(P, cin, cout, lin, stride, res_mode, KIND_TC, iters, ms_out);
}

int hb_op_stem_q(const void* xn, int P, int L, const float* w_host, const float* b_host, int cout, void* out,
                 int out_q, void* stream) {
  if (init_kernels() != cudaSuccess) return fail(nullptr, HB_E_CUDA, "kernel attribute setup failed");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int tot = kTaps - 1;
  float *dw = nullptr, *db = nullptr;
  hb_ctx* none = nullptr;
  CK(none, cudaMalloc(&dw, sizeof(float) * cout * kTaps));
  CK(none, cudaMemcpy(dw, w_host, sizeof(float) * cout * kTaps, cudaMemcpyHostToDevice));
  CK(none, cudaMalloc(&db, sizeof(float) * cout));
  CK(none, cudaMemcpy(db, b_host, sizeof(float) * cout, cudaMemcpyHostToDevice));
  // the stem's TMA view needs 16-B aligned rows: stage the [P][L] windows with a padded stride
  const int Lp = round_up(L, 8);
  __half* xp = nullptr;
  CK(none, cudaMalloc(&xp, sizeof(__half) * P * Lp));
  CK(none, cudaMemcpy2DAsync(xp, sizeof(__half) * Lp, xn, sizeof(__half) * L, sizeof(__half) * L, P,
                             cudaMemcpyDeviceToDevice, st));
  const StemMember sm{xp, dw, db};
  cudaError_t ce = launch_stem(&sm, 1, Lp, P, L, out_q, cout, tot / 2, static_cast<__half*>(out), st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
  cudaFree(dw);
  cudaFree(db);
  cudaFree(xp);
  if (ce != cudaSuccess) return fail(none, HB_E_CUDA, cudaGetErrorString(ce));
  return HB_OK;
}

int hb_op_stem(const void* xn, int P, int L, const float* w_host, const float* b_host, int cout, void* out,
               void* stream) {
  return hb_op_stem_q(xn, P, L, w_host, b_host, cout, out, 1, stream);
}

}  // extern "C"
