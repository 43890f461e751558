// Host-side orchestration of the level-by-level factorize / solve / matvec.
//
// A tree level is one batch: every per-node numpy call of the reference
// (solver.py:128-161, 210-253; treecode.py:76-127) becomes a descriptor in
// a level-wide launch.  Descriptor programs are built once per plan (and per
// right-hand-side count for solve / hmatvec) with relocatable operands
// (common.cuh: Ref / Bases), so a call only supplies base pointers.
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <vector>

#include "hks_internal.h"

namespace hks {

// Base-table slots beyond the HKS_BUF_* ids.
// B_XIN / B_XOUT: the shard-root exchange vectors of a sharded tree's
// subtree plan (HKS_PLAN_SUBTREE): r_0 x k blocks, ld r_0.
enum BaseSlot { B_FWS = HKS_NBUF, B_VIN, B_VOUT, B_VWS, B_XIN, B_XOUT };
static_assert(B_XOUT < kAbs, "base slots overflow");
static_assert(B_VWS == kGeconScratchBase, "gecon scratch base slot");

// Plan modes (hks_plan_create_ex).  A sharded tree is one subtree plan per
// rank (the rank's shard, rooted at a level-p node that still has a
// skeleton, Theta and a push) plus a top plan over levels 0..p whose leaves
// are the 2^p shard roots, supplied from outside (Theta, skeleton indices,
// up-pass vectors) instead of being factored.
enum PlanMode { PM_FULL = 0, PM_SUBTREE = 1, PM_TOP = 2 };

struct Layout {
  int64_t n = 0, depth = 0, nn = 0, s = 0;
  int mode = PM_FULL;
  // node i carries a skeleton (interp, Theta, push / phi): every node but
  // the root of a full or top tree
  bool has_up(int64_t i) const { return i > 0 || mode == PM_SUBTREE; }
  // leaves of a top plan are shard roots owned by other plans
  bool external(int64_t i) const { return mode == PM_TOP && is_leaf(i); }
  std::vector<int64_t> begin, size, rcap, ccap;
  std::vector<int64_t> off[HKS_NBUF];
  int64_t total[HKS_NBUF] = {0};

  bool is_leaf(int64_t i) const { return i >= ((int64_t)1 << depth) - 1; }
  int64_t first(int64_t level) const { return ((int64_t)1 << level) - 1; }
  int64_t count(int64_t level) const { return (int64_t)1 << level; }
};

Layout make_layout(int64_t n, int64_t depth, int64_t max_rank, int mode = PM_FULL);

enum StepKind {
  ST_GEMM, ST_COPY, ST_GETRF, ST_GETRS, ST_GECON, ST_EVAL_CM, ST_EVAL_RM, ST_KSUM,
  ST_PANEL, ST_SWAP, ST_TRSM_L, ST_TRSM_U, ST_NORM1, ST_LU_FUSED, ST_GATHER, ST_GETRS_FUSED,
  ST_FORK, ST_JOIN  // stream control: the side stream waits for / rejoins the main stream
};

struct Step {
  int kind;
  const void* d;  // device descriptors
  int count;
  int p0, p1;     // grid sizing (max dims)
  double flops;   // algorithmic FP64 flops of the whole step
  double bytes;   // compulsory HBM bytes of the whole step
  int stream;     // 0 main, 1 side (between ST_FORK and ST_JOIN)
};

constexpr int kNumKinds = 16;

// Opt-in per-kind CUDA-event timing of every step (hks_profile_*).
void profile_step(int kind, double flops, double bytes, cudaEvent_t a, cudaEvent_t b);
bool profiling();
void count_launch(int n = 1);

// Accumulates host descriptor arrays, uploads them in one arena.
class StepList {
 public:
  template <class D>
  void add(int kind, const std::vector<D>& v, int p0, int p1 = 0, double flops = 0.0, double bytes = 0.0) {
    if (v.empty()) return;
    size_t at = (host_.size() + 63) & ~size_t(63);
    host_.resize(at + v.size() * sizeof(D));
    std::memcpy(host_.data() + at, v.data(), v.size() * sizeof(D));
    offs_.push_back(at);
    steps_.push_back(Step{kind, nullptr, (int)v.size(), p0, p1, flops, bytes, side_now_ ? 1 : 0});
  }
  // Steps added between fork() and join() may run on the side stream
  // (side(true)) concurrently with main-stream steps added meanwhile;
  // join() makes the main stream wait for everything the side stream has.
  void fork() { control(ST_FORK); }
  void join() { control(ST_JOIN); }
  void side(bool on) { side_now_ = on; }
  cudaError_t upload(cudaStream_t stream);
  // ev (optional): marks().size() + 1 events, recorded before each marked
  // step and after the last step (per-level device timing)
  cudaError_t run(const Bases* dev_b, const double* X, int d, const KernelParams& kp, cudaStream_t stream,
                  cudaEvent_t* ev = nullptr, bool capturing = false) const;
  void mark() { marks_.push_back(steps_.size()); }
  const std::vector<size_t>& marks() const { return marks_; }
  void clear();
  StepList() = default;
  StepList(const StepList&) = delete;
  StepList& operator=(const StepList&) = delete;
  ~StepList();
  bool empty() const { return steps_.empty(); }
  size_t launches() const {
    size_t n = 0;
    for (auto& s : steps_) n += (s.kind != ST_FORK && s.kind != ST_JOIN);
    return n;
  }

 private:
  void control(int kind) {
    offs_.push_back(0);
    steps_.push_back(Step{kind, nullptr, 0, 0, 0, 0.0, 0.0, 0});
  }
  bool side_now_ = false;
  mutable cudaStream_t side_ = nullptr;
  mutable cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
  std::vector<char> host_;
  std::vector<size_t> offs_;
  std::vector<Step> steps_;
  std::vector<size_t> marks_;
  char* dev_ = nullptr;
  size_t dev_bytes_ = 0;
};

// Device scratch owned by a plan.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t b);
  ~DevBuf();
};

// Executable form of one StepList: a fixed device base table (the kernels
// read their operand bases from it, so a captured graph stays valid while
// the factor / vector buffers change between calls), a pinned ring that
// feeds it, and the CUDA graph captured on first use.
struct GraphCache {
  static constexpr int kRing = 16;
  Bases* dev = nullptr;
  Bases* host = nullptr;
  cudaEvent_t ring_ev[kRing] = {};
  int next = 0;
  cudaGraphExec_t exec = nullptr;
  bool with_memset = false;
  cudaStream_t cs = nullptr;
  cudaError_t write(const Bases& b, cudaStream_t s);
  ~GraphCache();
};

bool graphs_enabled();
bool node_priorities();  // graph nodes keep their capture stream's priority (plan.cu)

// Runs `sl` with bases `b` on stream s (graph replay unless profiling or
// HKS_GRAPHS=0); `memset_ptr` (if any) is zeroed first, inside the graph.
cudaError_t run_graphed(GraphCache& gc, const StepList& sl, const Bases& b, const double* X, int d,
                        const KernelParams& kp, cudaStream_t s, cudaEvent_t* ev, void* memset_ptr,
                        size_t memset_bytes, bool allow_graph = true);

struct VecProgram {
  StepList steps;
  DevBuf ws;
  GraphCache graphs;
  // subtree plans: the downward half (after the shard-root exchange),
  // sharing `ws` with the upward half in `steps`
  StepList down;
  GraphCache down_graphs;
};

}  // namespace hks

struct hks_plan {
  hks::Layout L;
  const double* X = nullptr;
  int64_t d = 0;
  std::vector<int64_t> rank;
  hks::KernelParams kp{};
  hks_kernel kern{};

  // cached leaf blocks K_aa (no lam), column-major m x m each (treecode.py:
  // 48-51 caches them too): hks_plan_cache_leaves.  Factorize then copies
  // K_aa + lam I into the LU storage and hmatvec's leaf level is a GEMM,
  // instead of evaluating the kernel every call.
  hks::DevBuf leaf_cache;
  std::vector<int64_t> leaf_off;            // element offset of each leaf's block (by heap index)
  bool leaf_cached = false;
  hks::StepList coup_steps;                 // build_operator
  hks::GraphCache coup_exec;
  std::unique_ptr<hks::StepList> fact[2];   // factorize without / with the anorm steps for dgecon
  hks::GraphCache fact_graphs[2];
  // dgecon estimates: one step per internal level, run on a side stream as
  // soon as that level's LU is done (waits on level_ev), never joined into
  // the factorization -- nothing downstream reads z_cond (solver.py:106).
  std::vector<std::unique_ptr<hks::StepList>> cond_levels;
  std::vector<int> cond_wait;               // level_ev index each cond level waits for
  cudaStream_t cond_stream = nullptr;       // caller's stream (hks_set_cond_stream) or own_cond_stream
  cudaStream_t own_cond_stream = nullptr;
  cudaEvent_t cond_done = nullptr;
  hks::GraphCache cond_gc;                  // device base table (+ pinned ring) of the cond launches
  bool cond_pending = false;
  hks::DevBuf fws;                          // factorize level workspace
  hks::DevBuf cond_ws;                      // dgecon state of the split estimate
  // factorize / solve / hmatvec programs run on a plan-owned high-priority
  // stream (joined to and from the caller's), so the low-priority dgecon
  // estimates only take SMs the level programs leave idle
  cudaStream_t hi = nullptr;
  cudaEvent_t hi_in = nullptr, hi_out = nullptr;
  std::vector<cudaEvent_t> level_ev;        // per-level factorize timing (leaf level first)
  std::map<int64_t, std::unique_ptr<hks::VecProgram>> solve_prog, mv_prog, up_prog;

  // stacked per-internal-node slots: node p owns R_p rows (x k columns);
  // a subtree plan's root owns r_0 more rows at root_slot
  std::vector<int64_t> stack_off;
  int64_t stack_total = 0;
  int64_t root_slot = -1;

  int64_t R(int64_t i) const { return rank[2 * i + 1] + rank[2 * i + 2]; }
  ~hks_plan() {
    if (cond_done) cudaEventSynchronize(cond_done);
    for (auto e : level_ev) cudaEventDestroy(e);
    if (cond_done) cudaEventDestroy(cond_done);
    if (own_cond_stream) cudaStreamDestroy(own_cond_stream);
    if (hi) cudaStreamDestroy(hi);
    if (hi_in) cudaEventDestroy(hi_in);
    if (hi_out) cudaEventDestroy(hi_out);
  }
};
