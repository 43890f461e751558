// Level-batched factorize / solve / hmatvec over the flat layout
// (solver.py:111-270, treecode.py:41-128) and the plan-bound C-ABI entry
// points.  See plan.h.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>

#include "plan.h"

namespace hks {

Layout make_layout(int64_t n, int64_t depth, int64_t s, int mode) {
  Layout L;
  L.n = n;
  L.depth = depth;
  L.s = s;
  L.mode = mode;
  L.nn = ((int64_t)1 << (depth + 1)) - 1;
  L.begin.assign(L.nn, 0);
  L.size.assign(L.nn, 0);
  L.rcap.assign(L.nn, 0);
  L.ccap.assign(L.nn, 0);
  L.size[0] = n;
  for (int64_t i = 0; i < L.first(depth); ++i) {  // tree.py:117,121: left takes ceil
    const int64_t half = (L.size[i] + 1) / 2;
    L.begin[2 * i + 1] = L.begin[i];
    L.size[2 * i + 1] = half;
    L.begin[2 * i + 2] = L.begin[i] + half;
    L.size[2 * i + 2] = L.size[i] - half;
  }
  for (int64_t i = L.nn - 1; i >= 0; --i) {
    L.ccap[i] = L.is_leaf(i) ? L.size[i] : L.rcap[2 * i + 1] + L.rcap[2 * i + 2];
    if (L.external(i)) L.rcap[i] = s;  // a shard root: rank <= s
    else L.rcap[i] = L.has_up(i) ? std::min<int64_t>(s, L.ccap[i]) : 0;
  }
  for (int b = 0; b < HKS_NBUF; ++b) L.off[b].assign(L.nn, -1);
  auto put = [&](int b, int64_t i, int64_t elems) {
    L.off[b][i] = L.total[b];
    L.total[b] += elems;
  };
  if (mode == PM_TOP)  // shard roots first, s x s / s apart: the exchange gathers straight into them
    for (int64_t i = L.first(depth); i < L.nn; ++i) {
      put(HKS_BUF_THETA, i, s * s);
      put(HKS_BUF_SKEL, i, s);
    }
  for (int64_t i = 0; i < L.nn; ++i) {
    L.off[HKS_BUF_STATS][i] = i;
    if (L.external(i)) continue;
    const bool leaf = L.is_leaf(i), up = L.has_up(i);
    if (up) {
      put(HKS_BUF_INTERP, i, L.rcap[i] * L.ccap[i]);
      put(HKS_BUF_SKEL, i, L.rcap[i]);
      put(HKS_BUF_THETA, i, L.rcap[i] * L.rcap[i]);
    }
    if (leaf) {
      put(HKS_BUF_LEAF_LU, i, L.size[i] * L.size[i]);
      put(HKS_BUF_LEAF_PIV, i, 4 * L.size[i]);  // pivots | total perm | panel perm | group perm
      if (up) put(HKS_BUF_PHI, i, L.size[i] * L.rcap[i]);
    } else {
      put(HKS_BUF_Z_LU, i, L.ccap[i] * L.ccap[i]);
      put(HKS_BUF_Z_PIV, i, 4 * L.ccap[i]);  // pivots | total perm | panel perm | group perm
      if (up) put(HKS_BUF_PUSH, i, L.ccap[i] * L.rcap[i]);
      put(HKS_BUF_COUP, i, L.rcap[2 * i + 1] * L.rcap[2 * i + 2]);
    }
  }
  L.total[HKS_BUF_STATS] = 3 * L.nn;
  return L;
}

cudaError_t StepList::upload(cudaStream_t stream) {
  if (host_.empty()) return cudaSuccess;
  if (dev_bytes_ < host_.size()) {
    if (dev_) cudaFree(dev_);
    dev_ = nullptr;
    cudaError_t e = cudaMalloc(&dev_, host_.size());
    if (e != cudaSuccess) return e;
    dev_bytes_ = host_.size();
  }
  cudaError_t e = cudaMemcpyAsync(dev_, host_.data(), host_.size(), cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  for (size_t s = 0; s < steps_.size(); ++s) steps_[s].d = dev_ + offs_[s];
  return e;
}

StepList::~StepList() {
  if (dev_) cudaFree(dev_);
  if (side_) cudaStreamDestroy(side_);
  if (fork_ev_) cudaEventDestroy(fork_ev_);
  if (join_ev_) cudaEventDestroy(join_ev_);
}

void StepList::clear() {
  host_.clear();
  offs_.clear();
  steps_.clear();
  marks_.clear();
}



cudaError_t DevBuf::ensure(size_t b) {
  if (b <= bytes) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
  cudaError_t e = cudaMalloc(&p, b);
  if (e == cudaSuccess) bytes = b;
  return e;
}

DevBuf::~DevBuf() {
  if (p) cudaFree(p);
}

cudaError_t StepList::run(const Bases* b, const double* X, int d, const KernelParams& kp,
                          cudaStream_t s, cudaEvent_t* ev, bool capturing) const {
  auto record = [&](cudaEvent_t e, cudaStream_t st) {
    if (capturing) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
  };
  const bool prof = profiling();
  size_t next_mark = 0;
  const cudaStream_t main = s;
  for (size_t si = 0; si < steps_.size(); ++si) {
    const Step& st = steps_[si];
    while (ev && next_mark < marks_.size() && marks_[next_mark] == si) record(ev[next_mark++], main);
    if (st.kind == ST_FORK || st.kind == ST_JOIN) {
      if (!side_) {
        // side branches (work nothing on the main chain waits for soon):
        // a priority between the main chain's and the dgecon stream's
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cudaError_t e = cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking,
                                                     node_priorities() ? (lo + hi) / 2 : 0);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
      }
      cudaError_t e = st.kind == ST_FORK ? cudaEventRecord(fork_ev_, main) : cudaEventRecord(join_ev_, side_);
      if (e == cudaSuccess)
        e = st.kind == ST_FORK ? cudaStreamWaitEvent(side_, fork_ev_, 0) : cudaStreamWaitEvent(main, join_ev_, 0);
      if (e != cudaSuccess) return e;
      continue;
    }
    s = st.stream ? side_ : main;
    cudaError_t e = cudaSuccess;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (prof) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
    count_launch();
    switch (st.kind) {
      case ST_GEMM:
        e = launch_gemm_batched(b, (const GemmDesc*)st.d, st.count, st.p0, st.p1, s);
        break;
      case ST_COPY:
        e = launch_copy_batched(b, (const CopyDesc*)st.d, st.count, st.p0, s);
        break;
      case ST_GETRF:
        e = launch_getrf_batched(b, (const LuDesc*)st.d, st.count, st.p0, s);
        break;
      case ST_GETRS:
        e = launch_getrs_batched(b, (const LuSolveDesc*)st.d, st.count, st.p0, st.p1, s);
        break;
      case ST_GECON:  // p1 = 0: one launch; p1 = 1 + phase: a step of the split estimate
        e = launch_gecon_batched(b, (const LuDesc*)st.d, st.count, st.p0, s, st.p1 - 1);
        break;
      case ST_EVAL_CM:
      case ST_EVAL_RM:
        e = launch_eval_batched(X, d, kp, b, (const EvalDesc*)st.d, st.count, st.p0, st.p1,
                                st.kind == ST_EVAL_RM, s);
        break;
      case ST_KSUM:
        e = launch_ksum_batched(X, d, kp, b, (const SumDesc*)st.d, st.count, st.p0, s);
        break;
      case ST_PANEL:
        e = launch_panel_batched(b, (const PanelDesc*)st.d, st.count, st.p0, st.p1, s);
        break;
      case ST_SWAP:
        e = launch_swap_batched(b, (const SwapDesc*)st.d, st.count, st.p0, s);
        break;
      case ST_GATHER:
        e = launch_gather_batched(b, (const GatherDesc*)st.d, st.count, st.p0, st.p1, s);
        break;
      case ST_GETRS_FUSED:
        e = launch_getrs_fused(b, (const GetrsDesc*)st.d, st.count, st.p0, st.p1, s);
        break;
      case ST_TRSM_L:
      case ST_TRSM_U:
        e = launch_trsm_batched(b, (const TrsmDesc*)st.d, st.count, st.p0, st.p1, st.kind == ST_TRSM_U, s);
        break;
      case ST_NORM1:
        e = launch_norm1_batched(b, (const LuDesc*)st.d, st.count, s);
        break;
      case ST_LU_FUSED:
        e = launch_lu_fused(b, (const LuFusedDesc*)st.d, st.count, st.p0, st.p1, s);
        break;
    }
    if (prof) {
      cudaEventRecord(e1, s);
      profile_step(st.kind, st.flops, st.bytes, e0, e1);
    }
    if (e != cudaSuccess) return e;
  }
  s = main;
  while (ev && next_mark < marks_.size()) record(ev[next_mark++], s);
  if (ev) record(ev[marks_.size()], s);
  return cudaSuccess;
}

// ------------------------------------------------------------ profiling

namespace {
struct Pending {
  int kind;
  double flops, bytes;
  cudaEvent_t a, b;
};
struct Profile {
  bool on = false;
  std::vector<Pending> pending;
  double launches[kNumKinds] = {0}, ms[kNumKinds] = {0}, flops[kNumKinds] = {0}, bytes[kNumKinds] = {0};
};
Profile g_prof;
long long g_launches = 0;
}  // namespace

bool profiling() { return g_prof.on; }
bool graphs_enabled() {
  static const int on = [] {
    const char* v = getenv("HKS_GRAPHS");
    return v ? atoi(v) : 1;
  }();
  return on != 0;
}

GraphCache::~GraphCache() {
  if (exec) cudaGraphExecDestroy(exec);
  if (cs) cudaStreamDestroy(cs);
  for (auto& e : ring_ev)
    if (e) cudaEventDestroy(e);
  if (host) cudaFreeHost(host);
  if (dev) cudaFree(dev);
}

cudaError_t GraphCache::write(const Bases& b, cudaStream_t s) {
  if (!dev) {
    cudaError_t e = cudaMalloc(&dev, sizeof(Bases));
    if (e == cudaSuccess) e = cudaMallocHost(&host, kRing * sizeof(Bases));
    for (int i = 0; i < kRing && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ring_ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  const int slot = next;
  next = (next + 1) % kRing;
  cudaError_t e = cudaEventSynchronize(ring_ev[slot]);  // the copy that last read this slot has run
  if (e != cudaSuccess) return e;
  host[slot] = b;
  e = cudaMemcpyAsync(dev, host + slot, sizeof(Bases), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaEventRecord(ring_ev[slot], s);
  return e;
}

// Graph nodes keep the priority of the stream they were captured on (main
// chain highest, side branches lower) when instantiated with
// cudaGraphInstantiateFlagUseNodePriority (HKS_NODE_PRIO=0: off).
bool node_priorities() {
  static const bool v = [] {
    const char* e = getenv("HKS_NODE_PRIO");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

cudaError_t run_graphed(GraphCache& gc, const StepList& sl, const Bases& b, const double* X, int d,
                        const KernelParams& kp, cudaStream_t s, cudaEvent_t* ev, void* memset_ptr,
                        size_t memset_bytes, bool allow_graph) {
  static const bool htrace = getenv("HKS_HOST_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = gc.write(b, s);
  if (htrace)
    fprintf(stderr, "HKS_HOST graph write %lld us\n",
            (long long)std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0)
                .count());
  if (e != cudaSuccess) return e;
  if (!allow_graph || !graphs_enabled() || profiling()) {
    e = memset_ptr ? cudaMemsetAsync(memset_ptr, 0, memset_bytes, s) : cudaSuccess;
    return e == cudaSuccess ? sl.run(gc.dev, X, d, kp, s, ev) : e;
  }
  if (!gc.exec) {  // capture once: the graph reads its bases from gc.dev
    if (!gc.cs) {  // captured at the highest priority (the nodes keep it: per-node priorities below)
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      e = cudaStreamCreateWithPriority(&gc.cs, cudaStreamNonBlocking, node_priorities() ? hi : 0);
      if (e != cudaSuccess) return e;
    }
    e = cudaStreamBeginCapture(gc.cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    cudaError_t er = sl.run(gc.dev, X, d, kp, gc.cs, ev, true);
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(gc.cs, &g);
    if (er != cudaSuccess) e = er;
    if (e == cudaSuccess)
      e = cudaGraphInstantiate(&gc.exec, g, node_priorities() ? cudaGraphInstantiateFlagUseNodePriority : 0);
    if (g) cudaGraphDestroy(g);
    if (e != cudaSuccess) return e;
  } else {
    count_launch((int)sl.launches());
  }
  if (memset_ptr) {
    e = cudaMemsetAsync(memset_ptr, 0, memset_bytes, s);
    if (e != cudaSuccess) return e;
  }
  return cudaGraphLaunch(gc.exec, s);
}

void count_launch(int n) { g_launches += n; }
void profile_step(int kind, double flops, double bytes, cudaEvent_t a, cudaEvent_t b) {
  g_prof.pending.push_back(Pending{kind, flops, bytes, a, b});
}

namespace {

inline Ref D(int buf, int64_t elem) { return make_ref(buf, (uint64_t)elem * 8); }
inline Ref I32(int buf, int64_t elem) { return make_ref(buf, (uint64_t)elem * 4); }
inline Ref adv(Ref r, int64_t elems) { return r + (uint64_t)elems * 8; }

struct Gemms {
  std::vector<GemmDesc> v;
  int mm = 0, mn = 0;
  double flops = 0, bytes = 0;
  void add(Ref A, int lda, int ta, Ref B, int ldb, int tb, Ref C, int ldc, int m, int n, int k,
           double alpha, double beta) {
    if (m <= 0 || n <= 0) return;
    v.push_back(GemmDesc{A, B, C, m, n, k, lda, ldb, ldc, ta, tb, alpha, beta});
    mm = std::max(mm, m);
    mn = std::max(mn, n);
    flops += 2.0 * m * n * k;
    bytes += 8.0 * ((double)m * k + (double)k * n + (double)m * n * (beta != 0.0 ? 2 : 1));
  }
  void flush(StepList& sl) {
    sl.add(ST_GEMM, v, mm, mn, flops, bytes);
    v.clear();
    mm = mn = 0;
    flops = bytes = 0;
  }
};

inline double lu_flops(double n) { return 2.0 / 3.0 * n * n * n; }
struct Copies {
  std::vector<CopyDesc> v;
  int me = 0;
  void copy(Ref src, int lds, int trans, Ref dst, int ldd, int m, int n) {
    if (m <= 0 || n <= 0) return;
    v.push_back(CopyDesc{src, dst, m, n, lds, ldd, trans, 0, 1.0});
    me = std::max(me, m * n);
  }
  // dst = lam * src (lam: the call's Bases::lam)
  void lam_scale(Ref src, int lds, Ref dst, int ldd, int m, int n) {
    if (m <= 0 || n <= 0) return;
    v.push_back(CopyDesc{src, dst, m, n, lds, ldd, 0, 5, 1.0});
    me = std::max(me, m * n);
  }
  // dst = src + lam I (lam: the call's Bases::lam)
  void add_lam_diag(Ref src, int lds, Ref dst, int ldd, int m, int n) {
    if (m <= 0 || n <= 0) return;
    v.push_back(CopyDesc{src, dst, m, n, lds, ldd, 0, 6, 1.0});
    me = std::max(me, m * n);
  }
  // dst = src^T + alpha * src2 (dst, src2: m x n; src: n x m)
  void transpose_add(Ref src, int lds, Ref src2, int lds2, Ref dst, int ldd, int m, int n, double alpha) {
    if (m <= 0 || n <= 0) return;
    v.push_back(CopyDesc{src, dst, m, n, lds, ldd, 1, 4, alpha, src2, lds2, 0});
    me = std::max(me, m * n);
  }
  void fill(Ref dst, int ldd, int m, int n, bool identity) {
    if (m <= 0 || n <= 0) return;
    v.push_back(CopyDesc{kNull, dst, m, n, 0, ldd, 0, identity ? 1 : 2, 1.0});
    me = std::max(me, m * n);
  }
  void flush(StepList& sl) {
    double bytes = 0;
    for (auto& c : v) bytes += (c.mode == 0 || c.mode >= 5 ? 16.0 : c.mode >= 3 ? 24.0 : 8.0) * c.m * c.n;
    sl.add(ST_COPY, v, me, 0, 0.0, bytes);
    v.clear();
    me = 0;
  }
};

struct Ctx {
  const hks_plan& P;
  const Layout& L;
  explicit Ctx(const hks_plan& p) : P(p), L(p.L) {}
  Ref interp(int64_t i) const { return D(HKS_BUF_INTERP, L.off[HKS_BUF_INTERP][i]); }
  Ref theta(int64_t i) const { return D(HKS_BUF_THETA, L.off[HKS_BUF_THETA][i]); }
  Ref leaf_lu(int64_t i) const { return D(HKS_BUF_LEAF_LU, L.off[HKS_BUF_LEAF_LU][i]); }
  Ref leaf_piv(int64_t i) const { return I32(HKS_BUF_LEAF_PIV, L.off[HKS_BUF_LEAF_PIV][i]); }
  Ref phi(int64_t i) const { return D(HKS_BUF_PHI, L.off[HKS_BUF_PHI][i]); }
  Ref z_lu(int64_t i) const { return D(HKS_BUF_Z_LU, L.off[HKS_BUF_Z_LU][i]); }
  Ref z_piv(int64_t i) const { return I32(HKS_BUF_Z_PIV, L.off[HKS_BUF_Z_PIV][i]); }
  // permutation workspace behind the pivots: [total | panel | group], `cap` ints each
  Ref leaf_ws(int64_t i) const { return I32(HKS_BUF_LEAF_PIV, L.off[HKS_BUF_LEAF_PIV][i] + L.size[i]); }
  Ref z_ws(int64_t i) const { return I32(HKS_BUF_Z_PIV, L.off[HKS_BUF_Z_PIV][i] + L.ccap[i]); }
  Ref push(int64_t i) const { return D(HKS_BUF_PUSH, L.off[HKS_BUF_PUSH][i]); }
  Ref coup(int64_t i) const { return D(HKS_BUF_COUP, L.off[HKS_BUF_COUP][i]); }
  Ref anorm(int64_t i) const { return D(HKS_BUF_STATS, i); }
  Ref rcond(int64_t i) const { return D(HKS_BUF_STATS, L.nn + i); }
  Ref info(int64_t i) const { return make_ref(HKS_BUF_STATS, (uint64_t)L.nn * 16 + (uint64_t)i * 4); }
  int r(int64_t i) const { return (int)P.rank[i]; }
  // stacked slot of node i inside its parent's R_p x k block (buffer `buf`, base element `at`)
  Ref slot(int buf, int64_t at, int64_t i, int64_t k, int* ld) const {
    if (i == 0) {  // root of a subtree plan: its own r_0 rows behind the internal nodes' blocks
      *ld = r(0);
      return D(buf, at + P.root_slot * k);
    }
    const int64_t p = (i - 1) / 2;
    *ld = (int)P.R(p);
    const int64_t row = (i == 2 * p + 1) ? 0 : P.rank[2 * p + 1];
    return D(buf, at + P.stack_off[p] * k + row);
  }
  Ref block(int buf, int64_t at, int64_t p, int64_t k) const { return D(buf, at + P.stack_off[p] * k); }
};

// ------------------------------------------------------------ LU programs

// One matrix of a level-batched LU: A (n x n, lda) factored in place with
// partial pivoting; optional right-hand sides B (n x r, ldb) carried through
// the factorization (forward substitution) and solved backward at the end,
// leaving B := A^-1 B (getrf + getrs, solver.py:131-135, 148-156).
struct LuJob {
  Ref A;
  int n, lda;
  Ref piv, info, anorm;
  Ref B;
  int r, ldb;
  Ref ws = kNull;  // int32 [total perm | panel perm | group perm], `cap` ints each (kNull: swap sweeps)
  int cap = 0;
  Ref Bsrc = kNull;  // add_lu_solve_program: right-hand sides read from here (ld ldb), B := A^-1 Bsrc
};

// Row permutations replace interchange sweeps for matrices up to this size
// (the register panel kernels track them; lu2.cu).
constexpr int kPermMaxRows = 1024;

struct Gathers {
  std::vector<GatherDesc> v;
  int mr = 0, mc = 0;
  void add(Ref A, int lda, Ref perm, int r0, int r1, int c0, int c1) {
    if (r1 - r0 <= 1 || c1 <= c0) return;
    v.push_back(GatherDesc{A, perm, lda, r0, r1, c0, c1, 0});
    mr = std::max(mr, r1 - r0);
    mc = std::max(mc, c1 - c0);
  }
  void flush(StepList& sl) {
    double bytes = 0;
    for (auto& d : v) bytes += 16.0 * (d.r1 - d.r0) * (d.c1 - d.c0);
    sl.add(ST_GATHER, v, mr, mc, 0.0, bytes);
    v.clear();
    mr = mc = 0;
  }
};

constexpr int kGroup = 128;  // rank of each trailing update (and TRSM block)

inline Ref elem(Ref base, int row, int col, int ld) { return adv(base, (int64_t)row + (int64_t)col * ld); }

struct Panels {
  std::vector<PanelDesc> v;
  int rows = 0;
  void flush(StepList& sl, int pb) {
    double f = 0;
    for (auto& d : v) f += (double)(d.n - d.p0) * d.pb * d.pb;
    sl.add(ST_PANEL, v, rows, pb, f, 0.0);
    v.clear();
    rows = 0;
  }
};

struct Swaps {
  std::vector<SwapDesc> v;
  int mc = 0;
  void add(Ref A, Ref piv, int lda, int r0, int r1, int c0, int c1) {
    if (r1 <= r0 || c1 <= c0) return;
    v.push_back(SwapDesc{A, piv, lda, r0, r1, c0, c1, 0});
    mc = std::max(mc, c1 - c0);
  }
  void flush(StepList& sl) {
    double bytes = 0;
    for (auto& d : v) bytes += 32.0 * (d.r1 - d.r0) * (d.c1 - d.c0);
    sl.add(ST_SWAP, v, mc, 0, 0.0, bytes);
    v.clear();
    mc = 0;
  }
};

struct Trsms {
  std::vector<TrsmDesc> v;
  int mc = 0, mk = 0;
  void add(Ref T, int ldt, Ref B, int ldb, int k, int ncols) {
    if (k <= 0 || ncols <= 0) return;
    v.push_back(TrsmDesc{T, B, ldt, ldb, k, ncols});
    mc = std::max(mc, ncols);
    mk = std::max(mk, k);
  }
  void flush(StepList& sl, bool upper) {
    double f = 0, bytes = 0;
    for (auto& d : v) {
      f += (double)d.k * d.k * d.ncols;
      bytes += 8.0 * ((double)d.k * d.k / 2 + 2.0 * d.k * d.ncols);
    }
    sl.add(upper ? ST_TRSM_U : ST_TRSM_L, v, mc, mk, f, bytes);
    v.clear();
    mc = mk = 0;
  }
};

// Appends the blocked, level-batched LU (+ carried right-hand sides) of
// `jobs` to `sl`.  Groups of 128 columns: 32-column panels (16 for n > 640)
// factored left-looking inside the group (swap, unit-lower TRSM and GEMM
// from the group's earlier panels), then the group's interchanges on every
// other column, one TRSM for the group's U rows and one rank-128 GEMM
// trailing update -- all matrices of the level in the same launches.
// Levels with at most this many matrices use the fused one-CTA-per-matrix
// LU (lu_fused.cu) instead of the multi-launch program (HKS_FUSED_MAX).
int fused_lu_max_count() {
  static const int v = [] {
    const char* e = getenv("HKS_FUSED_MAX");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// Panel width by the batch's largest matrix: the register panel kernels
// (lu2.cu) hold PB x rows/256 doubles per thread without spilling for
// 64 x 256, 32 x 512 and 16 x 1024.  Wider panels mean fewer in-group
// interchange / TRSM / GEMM steps per 128-column group.  HKS_PANEL_PB
// overrides (16, 32 or 64).
int panel_width(int nmax, int count) {
  static const int forced = [] {
    const char* e = getenv("HKS_PANEL_PB");
    return e ? atoi(e) : 0;
  }();
  static const int wide_count = [] {  // batches above this many matrices: 32-wide panels for <= 256 rows
    const char* e = getenv("HKS_PANEL32_COUNT");
    return e ? atoi(e) : 148;
  }();
  // 64 x 256 register panels run one CTA per SM (239 registers x 256
  // threads); a batch of more than one wave of them takes 32-wide panels
  // (two CTAs per SM) instead
  int pb = nmax <= 256 ? (count > wide_count ? 32 : 64) : nmax <= 512 ? 32 : 16;
  if (forced == 16 || forced == 32 || forced == 64) pb = forced;
  if (pb == 64 && nmax > 256) pb = 32;
  if (pb == 32 && nmax > 512) pb = 16;
  return pb;
}

// ||A||_1 of every matrix before it is factored (dgecon's anorm, solver.py:98).
void add_norm_step(StepList& sl, const std::vector<LuJob>& jobs) {
  std::vector<LuDesc> nd;
  int nmax = 0;
  for (auto& j : jobs) {
    nd.push_back(LuDesc{j.A, j.piv, j.info, j.anorm, kNull, j.n, j.lda});
    nmax = std::max(nmax, j.n);
  }
  sl.add(ST_NORM1, nd, nmax);
}

void add_lu_program(StepList& sl, const std::vector<LuJob>& jobs, bool with_norm) {
  if (jobs.empty()) return;
  int nmax = 0;
  for (auto& j : jobs) nmax = std::max(nmax, j.n);
  if (nmax == 0) return;
  const int PB = panel_width(nmax, (int)jobs.size());
  if (with_norm) add_norm_step(sl, jobs);
  if ((int)jobs.size() <= fused_lu_max_count()) {
    std::vector<LuFusedDesc> fd;
    double f = 0, bytes = 0;
    int rmax = 0;
    for (auto& j : jobs) {
      rmax = std::max(rmax, j.r);
      fd.push_back(LuFusedDesc{j.A, j.piv, j.info, j.r > 0 ? j.B : kNull, j.n, j.lda, j.r, j.ldb});
      f += lu_flops(j.n) + 2.0 * j.n * j.n * (double)j.r;
      bytes += 16.0 * ((double)j.n * j.n + (double)j.n * j.r);
    }
    sl.add(ST_LU_FUSED, fd, nmax, rmax, f, bytes);
    return;
  }
  // Interchanges: with permutation workspaces, one gather per pivot range
  // (the panel kernel records where every row went); otherwise LAPACK-style
  // sequential sweeps.  kind 0: this panel's pivots (rows from the panel's
  // first column), 1: the group's pivots so far (rows from g0).
  // Gathers over the panel/group permutations are slower than the pivot
  // sweeps on wide levels (many short CTAs) and faster on narrow ones; the
  // panels always record the total permutation (tperm) for the solves.
  bool track = nmax <= kPermMaxRows;
  for (auto& j : jobs) track &= j.ws != kNull;
  // measured (C2): gathers win for batches of <= 64 matrices (levels <= 6),
  // sweeps for the wide levels; HKS_LU_GATHER=0/1 forces either
  static const int gather_env = [] {
    const char* e = getenv("HKS_LU_GATHER");
    return e ? atoi(e) : -1;
  }();
  // (round 2, after the staged narrow-batch gathers: gathers also win on the
  // wide levels -- C3 124.7 -> 121.8 ms, C2 14.88 -> 14.77 ms -- so they are
  // the default whenever the permutations are recorded)
  const bool use_perm = track && (gather_env >= 0 ? gather_env != 0 : true);
  // The group-end interchanges (trailing columns and right-hand sides, the
  // wide ones) always gather by the group permutation when it is recorded:
  // one coalesced pass whatever the number of interchanges.  Sequential
  // sweeps are latency-serialised per interchange and ill-conditioned
  // blocks pivot almost every row (C3: 25 ms of sweeps per factorization).
  const bool gather_end = track && gather_env != 0;
  auto ws_perm = [](const LuJob& j, int which) { return j.ws + (uint64_t)which * j.cap * 4; };  // 0 total, 1 panel, 2 group
  struct Ix {
    Swaps sw;
    Gathers ga;
    void flush(StepList& sl) {
      sw.flush(sl);
      ga.flush(sl);
    }
  };
  auto interchange = [&](Ix& ix, const LuJob& j, Ref A, int lda, int kind, int r0, int r1, int c0, int c1,
                         bool group_end = false) {
    if (use_perm || (group_end && gather_end && kind == 1))
      ix.ga.add(A, lda, ws_perm(j, kind == 0 ? 1 : 2), r0, j.n, c0, c1);
    else
      ix.sw.add(A, j.piv, lda, r0, r1, c0, c1);
  };
  static const bool look_ahead = [] {
    const char* e = getenv("HKS_LOOKAHEAD");
    // round 1 measured it neutral; with the gathers above it hides the tail of
    // each trailing update behind the next group's panels (C3 -1.6 ms, C2 -0.3 ms)
    return e ? atoi(e) != 0 : true;
  }();
  bool side_pending = false;
  for (int g0 = 0; g0 < nmax; g0 += kGroup) {
    for (int p0 = g0; p0 < g0 + kGroup && p0 < nmax; p0 += PB) {
      Ix ix;
      Trsms tr;
      Gemms gm;
      Panels pn;
      for (auto& j : jobs) {
        if (p0 >= j.n) continue;
        const int gb = std::min(kGroup, j.n - g0), pb = std::min(PB, g0 + gb - p0);
        if (pb <= 0) continue;
        if (p0 > g0) {
          // previous panel's interchanges on the group's earlier L columns, and
          // all of the group's interchanges so far on this panel's columns
          const int q0 = p0 - PB;
          interchange(ix, j, j.A, j.lda, 0, q0, p0, g0, q0);
          interchange(ix, j, j.A, j.lda, 1, g0, p0, p0, p0 + pb);
          tr.add(elem(j.A, g0, g0, j.lda), j.lda, elem(j.A, g0, p0, j.lda), j.lda, p0 - g0, pb);
          gm.add(elem(j.A, p0, g0, j.lda), j.lda, 0, elem(j.A, g0, p0, j.lda), j.lda, 0, elem(j.A, p0, p0, j.lda),
                 j.lda, j.n - p0, pb, p0 - g0, -1.0, 1.0);
        }
        PanelDesc d{j.A, j.piv, j.info, j.lda, j.n, p0, pb, kNull, kNull, kNull, g0, 0};
        if (track) d.tperm = ws_perm(j, 0);
        if (gather_end) d.gperm = ws_perm(j, 2);
        if (use_perm) {
          d.tperm = ws_perm(j, 0);
          d.sig = ws_perm(j, 1);
          d.gperm = ws_perm(j, 2);
        }
        pn.v.push_back(d);
        pn.rows = std::max(pn.rows, j.n - p0);
      }
      ix.flush(sl);
      tr.flush(sl, false);
      gm.flush(sl);
      pn.flush(sl, PB);
    }
    // the group's interchanges everywhere else, U rows of the group, trailing
    // update.  Look-ahead: the next group's 128 columns are updated first on
    // the main stream, which then goes on to the next group's panels while
    // the rest of the trailing update (and the right-hand sides) runs on the
    // side stream; the next group end (whose interchanges touch this group's
    // L columns) joins it.
    if (side_pending) {
      sl.join();
      side_pending = false;
    }
    const bool ahead = look_ahead && g0 + 2 * kGroup < nmax + kGroup && g0 + kGroup < nmax;
    Ix ix;
    Trsms tr, tr_side;
    Gemms gm, gm_side;
    for (auto& j : jobs) {
      if (g0 >= j.n) continue;
      const int gb = std::min(kGroup, j.n - g0), ge = g0 + gb;
      const int last = g0 + ((gb - 1) / PB) * PB;  // first column of the group's last panel
      interchange(ix, j, j.A, j.lda, 0, last, ge, g0, last);
      interchange(ix, j, j.A, j.lda, 1, g0, ge, 0, g0, true);
      interchange(ix, j, j.A, j.lda, 1, g0, ge, ge, j.n, true);
      if (j.r > 0) interchange(ix, j, j.B, j.ldb, 1, g0, ge, 0, j.r, true);
      const int split = ahead ? std::min(j.n, ge + kGroup) : j.n;  // columns [ge, split) now, the rest later
      Trsms& tr2 = ahead ? tr_side : tr;
      Gemms& gm2 = ahead ? gm_side : gm;
      tr.add(elem(j.A, g0, g0, j.lda), j.lda, elem(j.A, g0, ge, j.lda), j.lda, gb, split - ge);
      gm.add(elem(j.A, ge, g0, j.lda), j.lda, 0, elem(j.A, g0, ge, j.lda), j.lda, 0, elem(j.A, ge, ge, j.lda), j.lda,
             j.n - ge, split - ge, gb, -1.0, 1.0);
      if (split < j.n) {
        tr2.add(elem(j.A, g0, g0, j.lda), j.lda, elem(j.A, g0, split, j.lda), j.lda, gb, j.n - split);
        gm2.add(elem(j.A, ge, g0, j.lda), j.lda, 0, elem(j.A, g0, split, j.lda), j.lda, 0,
                elem(j.A, ge, split, j.lda), j.lda, j.n - ge, j.n - split, gb, -1.0, 1.0);
      }
      if (j.r > 0) {
        tr2.add(elem(j.A, g0, g0, j.lda), j.lda, elem(j.B, g0, 0, j.ldb), j.ldb, gb, j.r);
        gm2.add(elem(j.A, ge, g0, j.lda), j.lda, 0, elem(j.B, g0, 0, j.ldb), j.ldb, 0, elem(j.B, ge, 0, j.ldb), j.ldb,
                j.n - ge, j.r, gb, -1.0, 1.0);
      }
    }
    ix.flush(sl);
    if (ahead) {
      sl.fork();
      sl.side(true);
      tr_side.flush(sl, false);
      gm_side.flush(sl);
      sl.side(false);
      side_pending = true;
    }
    tr.flush(sl, false);
    gm.flush(sl);
  }
  if (side_pending) sl.join();
  // backward: B := U^-1 B, groups from the bottom (right-looking)
  bool any_rhs = false;
  for (auto& j : jobs) any_rhs |= j.r > 0;
  if (!any_rhs) return;
  for (int g0 = ((nmax - 1) / kGroup) * kGroup; g0 >= 0; g0 -= kGroup) {
    Trsms tr;
    Gemms gm;
    for (auto& j : jobs) {
      if (j.r == 0 || g0 >= j.n) continue;
      const int gb = std::min(kGroup, j.n - g0);
      tr.add(elem(j.A, g0, g0, j.lda), j.lda, elem(j.B, g0, 0, j.ldb), j.ldb, gb, j.r);
      gm.add(elem(j.A, 0, g0, j.lda), j.lda, 0, elem(j.B, g0, 0, j.ldb), j.ldb, 0, j.B, j.ldb, g0, j.r, gb, -1.0, 1.0);
    }
    tr.flush(sl, true);
    gm.flush(sl);
  }
}

// B := A^-1 B with an LU from add_lu_program (getrs): interchanges, then
// unit-lower and upper sweeps in 128-row blocks (TRSM + GEMM updates).
void add_lu_solve_program(StepList& sl, const std::vector<LuJob>& jobs) {
  int nmax = 0;
  for (auto& j : jobs) nmax = std::max(nmax, j.n);
  if (nmax == 0) return;
  bool fused = nmax <= kGetrsFusedMax && getenv("HKS_GETRS_STEPS") == nullptr;
  for (auto& j : jobs) fused &= j.r == 0 || j.ws != kNull;
  if (fused) {  // one launch: gathered load, both sweeps (lu2.cu: getrs_fused_kernel)
    std::vector<GetrsDesc> v;
    int mc = 0;
    double f = 0, bytes = 0;
    for (auto& j : jobs) {
      if (j.r <= 0 || j.n <= 0) continue;
      v.push_back(GetrsDesc{j.A, j.ws, j.B, j.n, j.lda, j.ldb, j.r, 1, 0, j.Bsrc});
      mc = std::max(mc, j.r);
      f += 2.0 * j.n * j.n * (double)j.r;
      bytes += 8.0 * ((double)j.n * j.n + 2.0 * j.n * j.r);
    }
    sl.add(ST_GETRS_FUSED, v, nmax, mc, f, bytes);
    return;
  }
  Copies cs;  // separate sources: B := Bsrc first
  for (auto& j : jobs)
    if (j.r > 0 && j.Bsrc != kNull) cs.copy(j.Bsrc, j.ldb, 0, j.B, j.ldb, j.n, j.r);
  cs.flush(sl);
  Swaps sw;
  Gathers ga;
  for (auto& j : jobs) {
    if (j.r <= 0) continue;
    if (j.ws != kNull && j.n <= kPermMaxRows)
      ga.add(j.B, j.ldb, j.ws, 0, j.n, 0, j.r);  // total permutation recorded by the factorization
    else
      sw.add(j.B, j.piv, j.ldb, 0, j.n, 0, j.r);
  }
  sw.flush(sl);
  ga.flush(sl);
  for (int g0 = 0; g0 < nmax; g0 += kGroup) {
    Trsms tr;
    Gemms gm;
    for (auto& j : jobs) {
      if (j.r == 0 || g0 >= j.n) continue;
      const int gb = std::min(kGroup, j.n - g0), ge = g0 + gb;
      tr.add(elem(j.A, g0, g0, j.lda), j.lda, elem(j.B, g0, 0, j.ldb), j.ldb, gb, j.r);
      gm.add(elem(j.A, ge, g0, j.lda), j.lda, 0, elem(j.B, g0, 0, j.ldb), j.ldb, 0, elem(j.B, ge, 0, j.ldb), j.ldb,
             j.n - ge, j.r, gb, -1.0, 1.0);
    }
    tr.flush(sl, false);
    gm.flush(sl);
  }
  for (int g0 = ((nmax - 1) / kGroup) * kGroup; g0 >= 0; g0 -= kGroup) {
    Trsms tr;
    Gemms gm;
    for (auto& j : jobs) {
      if (j.r == 0 || g0 >= j.n) continue;
      const int gb = std::min(kGroup, j.n - g0);
      tr.add(elem(j.A, g0, g0, j.lda), j.lda, elem(j.B, g0, 0, j.ldb), j.ldb, gb, j.r);
      gm.add(elem(j.A, 0, g0, j.lda), j.lda, 0, elem(j.B, g0, 0, j.ldb), j.ldb, 0, j.B, j.ldb, g0, j.r, gb, -1.0, 1.0);
    }
    tr.flush(sl, true);
    gm.flush(sl);
  }
}

// dgecon scratch of the split estimate: every internal node x
// gecon_stride(max R) doubles (levels are batched into groups, below)
size_t cond_scratch_elems(const hks_plan& P) {
  int maxR = 0;
  for (int64_t i = 0; i < P.L.first(P.L.depth); ++i) maxR = std::max<int>(maxR, (int)P.R(i));
  return (size_t)std::max<int64_t>(P.L.first(P.L.depth), 1) * gecon_stride(maxR);
}

size_t factorize_workspace(const hks_plan& P) {
  size_t need = 0;
  for (int64_t lev = P.L.has_up(0) ? 0 : 1; lev < P.L.depth; ++lev) {
    size_t lv = 0;
    for (int64_t i = P.L.first(lev); i < P.L.first(lev) + P.L.count(lev); ++i) {
      const int64_t R = P.R(i);
      lv += 3 * R * P.rank[i];
    }
    need = std::max(need, lv);
  }
  return need;
}

// ------------------------------------------------------------ factorize

// The dgecon estimates of levels deeper than this start once the
// factorization has finished this level (HKS_COND_START_LEVEL overrides).
// Measured (C2, depth 9): starting the deep levels' chain at level 6 with at
// most 112 estimate CTAs (lu.cu) beats starting it at level 3 with one CTA
// per matrix (16.7 vs 16.9 ms); for deeper trees (C3, depth 11: ~2000
// matrices in the chain) the capped chain outlasts the factorization and
// level 3 with one CTA per matrix is best (152 vs 157 ms).
int64_t cond_start_level(int64_t depth) {
  static const int64_t forced = [] {
    const char* e = getenv("HKS_COND_START_LEVEL");
    return e ? (int64_t)atoi(e) : (int64_t)-1;
  }();
  if (forced >= 0) return forced;
  return depth <= 9 ? 6 : 3;
}

// Levels batched per estimate group: the estimate is a chain of
// kGeconSteps + 1 short launches whose length does not depend on the
// number of matrices, so one chain for all levels deeper than the start
// level and one for the levels above it (after the root) replaces one
// chain per level on the serial condition stream (HKS_COND_GROUPS=0: one
// group per level).
bool cond_grouped() {
  static const bool v = [] {
    const char* e = getenv("HKS_COND_GROUPS");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

void build_factorize(const hks_plan& P, bool with_cond, StepList& sl,
                     std::vector<std::unique_ptr<StepList>>* cond_levels, std::vector<int>* cond_wait) {
  const Ctx c(P);
  const Layout& L = P.L;
  // What the narrow top levels need that depends on no factor -- Z := I
  // (solver.py:145) -- in one side branch beside the leaf level (joined
  // before the first internal level): one fewer launch in each
  // latency-bound level.  Wide levels keep them in-level (their bytes
  // would compete with the leaf level's).
  bool early_pending = false;
  const int64_t early_levels = std::min<int64_t>(L.depth, 6);  // levels 0..5: <= 32 nodes
  auto early_node = [&](int64_t i) { return i < L.first(early_levels); };
  {
    Copies early;
    for (int64_t i = 0; i < L.first(early_levels); ++i) {
      const int rl = c.r(2 * i + 1), R = rl + c.r(2 * i + 2);
      // only Z's diagonal blocks: the coupling products below write the
      // off-diagonal ones (beta = 0), so they are neither zeroed nor re-read
      early.fill(c.z_lu(i), R, rl, rl, true);
      early.fill(adv(c.z_lu(i), (int64_t)rl * R + rl), R, R - rl, R - rl, true);
    }
    if (!early.v.empty()) {
      sl.fork();
      sl.side(true);
      early.flush(sl);
      sl.side(false);
      early_pending = true;
    }
  }
  sl.mark();
  if (L.mode != PM_TOP) {  // leaf level (solver.py:128-137): A = K + lam I, LU with P^T carried -> phi, theta = P phi
    std::vector<EvalDesc> ev;
    std::vector<LuJob> jobs;
    Copies cp;
    Gemms gm;
    int mx = 0;
    for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
      const int m = (int)L.size[i], r = L.has_up(i) ? c.r(i) : 0;
      if (P.leaf_cached)  // K_aa + lam I from the cached leaf block
        cp.add_lam_diag(abs_ref(static_cast<const double*>(P.leaf_cache.p) + P.leaf_off[i]), m, c.leaf_lu(i), m, m, m);
      else
        ev.push_back(EvalDesc{kNull, kNull, L.begin[i], L.begin[i], m, m, c.leaf_lu(i), m, 1});
      mx = std::max(mx, m);
      if (r > 0) cp.copy(c.interp(i), r, 1, c.phi(i), m, m, r);  // phi = P^T, then A^-1 P^T
      jobs.push_back(LuJob{c.leaf_lu(i), m, m, c.leaf_piv(i), c.info(i), kNull, r > 0 ? c.phi(i) : kNull, r, m,
                           c.leaf_ws(i), m});
      if (r > 0) gm.add(c.interp(i), r, 0, c.phi(i), m, 0, c.theta(i), r, r, r, m, 1.0, 0.0);
    }
    double ef = 0, eb = 0;
    for (auto& e : ev) {
      ef += (double)e.m * e.n * (2.0 * P.d + 5.0);
      eb += 8.0 * e.m * e.n;
    }
    sl.add(ST_EVAL_CM, ev, mx, mx, ef, eb);
    cp.flush(sl);
    add_lu_program(sl, jobs, false);
    gm.flush(sl);
  }
  std::vector<LuDesc> cond_group;  // estimates not yet emitted (see cond_grouped)
  int cond_maxR = 0;
  double cond_lb = 0;
  for (int64_t lev = L.depth - 1; lev >= 0; --lev) {  // internal levels (solver.py:139-161)
    sl.mark();
    if (early_pending) {
      sl.join();
      early_pending = false;
    }
    // Algebraically identical to solver.py:145-158 with the interpolation
    // folded in before the reduced solve: V = thhat P^T (R x r), Y = Z^-1 V,
    // F = B Y (= folded P^T), push = P^T - F, theta = P thhat push
    // (= P (thhat - thhat folded) P^T).  Solving for r instead of R
    // right-hand sides halves the node's flops; forming theta from push
    // needs V only once (as the LU's right-hand sides).
    Copies c_id, c_p;
    Gemms g_z, g_v, g_f, g_tf, g_out;
    std::vector<LuJob> jobs;
    std::vector<LuDesc> lu;
    int maxR = 0;
    int64_t at = 0;
    for (int64_t i = L.first(lev); i < L.first(lev) + L.count(lev); ++i) {
      const int64_t a = 2 * i + 1, b = 2 * i + 2;
      const int rl = c.r(a), rr = c.r(b), R = rl + rr, r = c.r(i);
      maxR = std::max(maxR, R);
      const Ref Z = c.z_lu(i), C = c.coup(i);
      if (!early_node(i)) {  // else the diagonal blocks come from the early branch
        c_id.fill(Z, R, rl, rl, true);
        c_id.fill(adv(Z, (int64_t)rl * R + rl), R, rr, rr, true);
      }
      g_z.add(c.theta(a), rl, 0, C, rl, 0, adv(Z, (int64_t)rl * R), R, rl, rr, rl, 1.0, 0.0);
      g_z.add(c.theta(b), rr, 0, C, rl, 1, adv(Z, rl), R, rr, rl, rr, 1.0, 0.0);
      lu.push_back(LuDesc{Z, c.z_piv(i), c.info(i), c.anorm(i), with_cond ? c.rcond(i) : kNull, R, R});
      if (!L.has_up(i)) {
        jobs.push_back(LuJob{Z, R, R, c.z_piv(i), c.info(i), c.anorm(i), kNull, 0, R, c.z_ws(i), (int)L.ccap[i]});
        continue;
      }
      const Ref Y = D(B_FWS, at);
      at += (int64_t)R * r;
      const Ref F = D(B_FWS, at);
      at += (int64_t)R * r;
      const Ref W = D(B_FWS, at);
      at += (int64_t)R * r;
      const Ref Pi = c.interp(i), pu = c.push(i);
      // V = thhat P^T into Y (the LU's right-hand sides)
      g_v.add(c.theta(a), rl, 0, Pi, r, 1, Y, R, rl, r, rl, 1.0, 0.0);
      g_v.add(c.theta(b), rr, 0, adv(Pi, (int64_t)rl * r), r, 1, adv(Y, rl), R, rr, r, rr, 1.0, 0.0);
      jobs.push_back(LuJob{Z, R, R, c.z_piv(i), c.info(i), c.anorm(i), Y, r, R, c.z_ws(i), (int)L.ccap[i]});  // Y = Z^-1 V
      // F = B Y (solver.py:86-89, 156); push = P^T - F (solver.py:158), one pass
      g_f.add(C, rl, 0, adv(Y, rl), R, 0, F, R, rl, r, rr, 1.0, 0.0);
      g_f.add(C, rl, 1, Y, R, 0, adv(F, rl), R, rr, r, rl, 1.0, 0.0);
      c_p.transpose_add(Pi, r, F, R, pu, R, R, r, -1.0);
      // W = thhat push ; theta = P W (solver.py:157)
      g_tf.add(c.theta(a), rl, 0, pu, R, 0, W, R, rl, r, rl, 1.0, 0.0);
      g_tf.add(c.theta(b), rr, 0, adv(pu, rl), R, 0, adv(W, rl), R, rr, r, rr, 1.0, 0.0);
      g_out.add(Pi, r, 0, W, R, 0, c.theta(i), r, r, r, R, 1.0, 0.0);
    }
    c_id.flush(sl);
    g_z.flush(sl);
    if (with_cond) {  // ||Z||_1 for dgecon (solver.py:98) beside V = thhat P^T, before Z is overwritten
      sl.fork();
      sl.side(true);
      add_norm_step(sl, jobs);
      sl.side(false);
    }
    g_v.flush(sl);
    if (with_cond) sl.join();
    add_lu_program(sl, jobs, false);
    if (with_cond && cond_levels) {
      for (auto& d : lu) cond_lb += 16.0 * d.n * d.n;
      cond_group.insert(cond_group.end(), lu.begin(), lu.end());
      cond_maxR = std::max(cond_maxR, maxR);
      // the estimates of levels deeper than cond_start_level wait until the
      // factorization reaches it: they then fill SMs the latency-bound top
      // levels leave idle instead of competing with the wide levels
      const int64_t start = cond_start_level(L.depth);
      if (!cond_grouped() || lev == 0 || lev == start) {
        cond_levels->emplace_back(new StepList());
        // split estimate: short-lived CTAs turn the SMs over to the
        // factorization's kernels between LU applications (lu.cu)
        for (int ph = 0; ph <= kGeconSteps; ++ph)
          cond_levels->back()->add(ST_GECON, cond_group, cond_maxR, 1 + ph, ph ? 2.0 * cond_lb / 16.0 : 0.0,
                                   ph ? cond_lb / 2.0 : 0.0);
        cond_wait->push_back((int)(L.depth - std::min<int64_t>(lev, start) + 1));
        cond_group.clear();
        cond_maxR = 0;
        cond_lb = 0;
      }
    }
    if (lev == 0 && !L.has_up(0)) continue;
    g_f.flush(sl);
    c_p.flush(sl);
    g_tf.flush(sl);
    g_out.flush(sl);
  }
}

// ------------------------------------------------------------ solve

// part: 0 the whole solve; subtree plans run it in two halves around the
// shard-root exchange -- 1 upward (psi of the root into B_XOUT), 2 downward
// (the root's incoming correction from B_XIN).  Top plans read the shard
// roots' psi from B_VIN and write their corrections to B_VOUT, shard j's
// r_j x k block at j * s * k (ld r_j).
void build_solve(const hks_plan& P, int64_t kk, int part, StepList& sl) {
  const Ctx c(P);
  const Layout& L = P.L;
  const int k = (int)kk, n = (int)L.n;
  const int64_t stk = P.stack_total * kk;
  const int64_t S = 0, G = stk, Gb = 2 * stk;  // element bases inside B_VWS
  const int64_t xs = L.s * kk;                  // top plans: shard-root block stride
  const bool sub = L.mode == PM_SUBTREE;
  bool forked = false;
  if (part != 2) {
    if (L.mode == PM_TOP) {  // shard roots: their psi arrive from the subtree plans
      Copies cp;
      for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
        int ld;
        const Ref dst = c.slot(B_VWS, S, i, k, &ld);
        cp.copy(D(B_VIN, (i - L.first(L.depth)) * xs), c.r(i), 0, dst, ld, c.r(i), k);
      }
      cp.flush(sl);
    } else {  // upward, leaves (solver.py:215-218)
      Gemms gp;
      Copies cp;
      std::vector<LuJob> jobs;
      int mx = 0;
      for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
        const int m = (int)L.size[i], r = c.r(i);
        mx = std::max(mx, m);
        if (L.has_up(i) && r > 0) {
          int ld;
          const Ref dst = c.slot(B_VWS, S, i, k, &ld);
          gp.add(c.phi(i), m, 1, D(B_VIN, L.begin[i]), n, 0, dst, ld, r, k, m, 1.0, 0.0);
        }
        cp.copy(D(B_VIN, L.begin[i]), n, 0, D(B_VOUT, L.begin[i]), n, m, k);
        jobs.push_back(LuJob{c.leaf_lu(i), m, m, c.leaf_piv(i), kNull, kNull, D(B_VOUT, L.begin[i]), k, n,
                             c.leaf_ws(i), m});
      }
      gp.flush(sl);
      // The leaf solves x = A^-1 b feed nothing until the final x -= phi c
      // (solver.py:215-217, 247-250): they run on the side stream while the
      // latency-bound internal levels run on the main one.
      forked = L.depth > 0 || sub;
      if (forked) {
        sl.fork();
        sl.side(true);
      }
      cp.flush(sl);
      add_lu_solve_program(sl, jobs);
      if (forked) sl.side(false);
    }
    for (int64_t lev = L.depth - 1; lev >= 0; --lev) {  // upward, internal (solver.py:219-233)
      Copies cp;
      std::vector<LuJob> jobs;
      Gemms g1, g2, g3;
      for (int64_t i = L.first(lev); i < L.first(lev) + L.count(lev); ++i) {
        const int64_t a = 2 * i + 1, bb = 2 * i + 2;
        const int rl = c.r(a), rr = c.r(bb), R = rl + rr, r = c.r(i);
        const Ref Si = c.block(B_VWS, S, i, k), Gi = c.block(B_VWS, G, i, k), Gbi = c.block(B_VWS, Gb, i, k);
        const Ref C = c.coup(i);
        // G = Z^-1 S (solver.py:222-226), S kept for the update below
        LuJob zj{c.z_lu(i), R, R, c.z_piv(i), kNull, kNull, Gi, k, R, c.z_ws(i), (int)L.ccap[i]};
        zj.Bsrc = Si;
        jobs.push_back(zj);
        g1.add(C, rl, 0, adv(Gi, rl), R, 0, Gbi, R, rl, k, rr, 1.0, 0.0);
        g1.add(C, rl, 1, Gi, R, 0, adv(Gbi, rl), R, rr, k, rl, 1.0, 0.0);
        if (!L.has_up(i)) continue;
        g2.add(c.theta(a), rl, 0, Gbi, R, 0, Si, R, rl, k, rl, -1.0, 1.0);
        g2.add(c.theta(bb), rr, 0, adv(Gbi, rl), R, 0, adv(Si, rl), R, rr, k, rr, -1.0, 1.0);
        int ld;
        const Ref dst = c.slot(B_VWS, S, i, k, &ld);
        g3.add(c.interp(i), r, 0, Si, R, 0, dst, ld, r, k, R, 1.0, 0.0);
      }
      cp.flush(sl);
      add_lu_solve_program(sl, jobs);
      g1.flush(sl);
      g2.flush(sl);
      g3.flush(sl);
    }
    if (sub) {  // psi of the shard root, for the top plan
      Copies cp;
      int ld;
      const Ref src_ = c.slot(B_VWS, S, 0, k, &ld);
      cp.copy(src_, ld, 0, D(B_XOUT, 0), c.r(0), c.r(0), k);
      cp.flush(sl);
    }
  }
  if (part == 1) {
    if (forked) sl.join();  // the down half is another program
    return;
  }
  if (sub) {  // the shard root's correction, from the top plan
    Copies cp;
    int ld;
    const Ref dst_ = c.slot(B_VWS, Gb, 0, k, &ld);
    cp.copy(D(B_XIN, 0), c.r(0), 0, dst_, ld, c.r(0), k);
    cp.flush(sl);
  }
  for (int64_t lev = sub ? 0 : 1; lev < L.depth; ++lev) {  // downward (solver.py:235-253)
    Gemms g;
    for (int64_t i = L.first(lev); i < L.first(lev) + L.count(lev); ++i) {
      const int R = (int)P.R(i), r = c.r(i);
      if (r == 0) continue;
      int ld;
      const Ref cin = c.slot(B_VWS, Gb, i, k, &ld);
      g.add(c.push(i), R, 0, cin, ld, 0, c.block(B_VWS, Gb, i, k), R, R, k, r, 1.0, 1.0);
    }
    g.flush(sl);
  }
  if (L.mode == PM_TOP) {  // corrections of the shard roots, for the subtree plans
    Copies cp;
    for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
      int ld;
      const Ref src_ = c.slot(B_VWS, Gb, i, k, &ld);
      cp.copy(src_, ld, 0, D(B_VOUT, (i - L.first(L.depth)) * xs), c.r(i), c.r(i), k);
    }
    cp.flush(sl);
  } else if (L.depth > 0 || sub) {
    if (forked) sl.join();
    Gemms g;
    for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
      const int m = (int)L.size[i], r = c.r(i);
      if (r == 0) continue;
      int ld;
      const Ref cin = c.slot(B_VWS, Gb, i, k, &ld);
      g.add(c.phi(i), m, 0, cin, ld, 0, D(B_VOUT, L.begin[i]), n, m, k, r, -1.0, 1.0);
    }
    g.flush(sl);
  }
}

// ------------------------------------------------------------ hmatvec / upward

void build_upward(const hks_plan& P, int64_t kk, int64_t S, StepList& sl) {
  const Ctx c(P);
  const Layout& L = P.L;
  const int k = (int)kk, n = (int)L.n;
  if (L.depth == 0 && !L.has_up(0)) return;
  Gemms g;
  Copies cp;
  for (int64_t i = L.first(L.depth); i < L.nn; ++i) {  // treecode.py:81-82
    int ld;
    const Ref dst = c.slot(B_VWS, S, i, k, &ld);
    if (L.external(i))  // a top plan's shard root: skeleton weights from its subtree plan
      cp.copy(D(B_VIN, (i - L.first(L.depth)) * L.s * kk), c.r(i), 0, dst, ld, c.r(i), k);
    else
      g.add(c.interp(i), c.r(i), 0, D(B_VIN, L.begin[i]), n, 0, dst, ld, c.r(i), k, (int)L.size[i], 1.0, 0.0);
  }
  g.flush(sl);
  cp.flush(sl);
  for (int64_t lev = L.depth - 1; lev >= (L.has_up(0) ? 0 : 1); --lev) {  // treecode.py:83-88
    Gemms g2;
    for (int64_t i = L.first(lev); i < L.first(lev) + L.count(lev); ++i) {
      int ld;
      const Ref dst = c.slot(B_VWS, S, i, k, &ld);
      const int R = (int)P.R(i);
      g2.add(c.interp(i), c.r(i), 0, c.block(B_VWS, S, i, k), R, 0, dst, ld, c.r(i), k, R, 1.0, 0.0);
    }
    g2.flush(sl);
  }
}

// part as in build_solve: subtree plans send the root's skeleton weights
// (B_XOUT) and receive its incoming accumulator (B_XIN); top plans read the
// shard roots' weights from B_VIN and write their accumulators to B_VOUT.
void build_matvec(const hks_plan& P, int64_t kk, int part, StepList& sl) {
  const Ctx c(P);
  const Layout& L = P.L;
  const int k = (int)kk, n = (int)L.n;
  const int64_t stk = P.stack_total * kk;
  const int64_t S = 0, A = stk;
  const bool sub = L.mode == PM_SUBTREE;
  if (part != 2) {
    if (L.mode != PM_TOP && P.leaf_cached) {  // leaves from the cached blocks: u = lam w, u += K_aa w
      Copies lw;
      Gemms g;
      for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
        const int m = (int)L.size[i];
        lw.lam_scale(D(B_VIN, L.begin[i]), n, D(B_VOUT, L.begin[i]), n, m, k);
        g.add(abs_ref(static_cast<const double*>(P.leaf_cache.p) + P.leaf_off[i]), m, 0, D(B_VIN, L.begin[i]), n, 0,
              D(B_VOUT, L.begin[i]), n, m, k, m, 1.0, 1.0);
      }
      lw.flush(sl);
      g.flush(sl);
    } else if (L.mode != PM_TOP) {  // leaves: u = K w + lam w, K never stored (treecode.py:99-101)
      std::vector<SumDesc> ks;
      int mx = 0;
      for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
        const int m = (int)L.size[i];
        mx = std::max(mx, m);
        ks.push_back(SumDesc{kNull, kNull, L.begin[i], L.begin[i], m, m, k, D(B_VIN, L.begin[i]), n,
                             D(B_VOUT, L.begin[i]), n, 0.0, 1});
      }
      double kf = 0, kb = 0;
      for (auto& q : ks) {
        kf += (double)q.m * q.n * (2.0 * P.d + 5.0) + 2.0 * q.m * q.n * q.k;
        kb += 8.0 * ((double)q.n * q.k + (double)q.m * q.k);
      }
      sl.add(ST_KSUM, ks, mx, 0, kf, kb);
    }
    if (L.depth == 0 && !sub) return;
    build_upward(P, kk, S, sl);
    if (sub) {
      Copies cp;
      int ld;
      const Ref src_ = c.slot(B_VWS, S, 0, k, &ld);
      cp.copy(src_, ld, 0, D(B_XOUT, 0), c.r(0), c.r(0), k);
      cp.flush(sl);
    }
  }
  if (part == 1) return;
  if (sub) {
    Copies cp;
    int ld;
    const Ref dst_ = c.slot(B_VWS, A, 0, k, &ld);
    cp.copy(D(B_XIN, 0), c.r(0), 0, dst_, ld, c.r(0), k);
    cp.flush(sl);
  }
  for (int64_t lev = 0; lev < L.depth; ++lev) {  // downward (treecode.py:109-123)
    Gemms gp, gc;
    for (int64_t i = L.first(lev); i < L.first(lev) + L.count(lev); ++i) {
      const int64_t a = 2 * i + 1, bb = 2 * i + 2;
      const int rl = c.r(a), rr = c.r(bb), R = rl + rr, r = c.r(i);
      const Ref Ai = c.block(B_VWS, A, i, k), Si = c.block(B_VWS, S, i, k), C = c.coup(i);
      const bool has_acc = L.has_up(i);
      if (has_acc) {
        int ld;
        const Ref acc = c.slot(B_VWS, A, i, k, &ld);
        gp.add(c.interp(i), r, 1, acc, ld, 0, Ai, R, R, k, r, 1.0, 0.0);
      }
      const double beta = has_acc ? 1.0 : 0.0;
      gc.add(C, rl, 0, adv(Si, rl), R, 0, Ai, R, rl, k, rr, 1.0, beta);
      gc.add(C, rl, 1, Si, R, 0, adv(Ai, rl), R, rr, k, rl, 1.0, beta);
    }
    gp.flush(sl);
    gc.flush(sl);
  }
  if (L.mode == PM_TOP) {
    Copies cp;
    for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
      int ld;
      const Ref src_ = c.slot(B_VWS, A, i, k, &ld);
      cp.copy(src_, ld, 0, D(B_VOUT, (i - L.first(L.depth)) * L.s * kk), c.r(i), c.r(i), k);
    }
    cp.flush(sl);
    return;
  }
  Gemms g;  // leaves (treecode.py:124-127)
  for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
    const int m = (int)L.size[i], r = c.r(i);
    if (r == 0) continue;
    int ld;
    const Ref acc = c.slot(B_VWS, A, i, k, &ld);
    g.add(c.interp(i), r, 1, acc, ld, 0, D(B_VOUT, L.begin[i]), n, m, k, r, 1.0, 1.0);
  }
  g.flush(sl);
}

}  // namespace
}  // namespace hks

// ======================================================================= C ABI

using namespace hks;

static inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

static Bases make_bases(void* const* buffers) {
  Bases b;
  std::memset(&b, 0, sizeof(b));
  for (int i = 0; i < HKS_NBUF; ++i) b.p[i] = buffers ? static_cast<char*>(buffers[i]) : nullptr;
  return b;
}

extern "C" int hks_layout(int64_t n, int64_t depth, int64_t max_rank, int64_t* sizes, int64_t* offsets) {
  if (n < 1 || depth < 0 || depth > 40 || max_rank < 1)
    return set_error(HKS_ERR_INVALID, "hks_layout: bad arguments n=%lld depth=%lld max_rank=%lld",
                     (long long)n, (long long)depth, (long long)max_rank);
  Layout L = make_layout(n, depth, max_rank);
  for (int b = 0; b < HKS_NBUF; ++b) {
    if (sizes) sizes[b] = L.total[b];
    if (offsets) std::memcpy(offsets + b * L.nn, L.off[b].data(), L.nn * sizeof(int64_t));
  }
  return HKS_OK;
}

// Dense LU / solve of one matrix through the same level programs the
// factorization uses (add_lu_program / add_lu_solve_program), so the dense
// entry points and the tree factorization share every kernel.
extern "C" int hks_lu_factor(double* A, int64_t n, int64_t lda, int32_t* piv, int32_t* info_host, void* stream) {
  if (n < 0 || lda < n) return set_error(HKS_ERR_INVALID, "hks_lu_factor: bad dims");
  if (n == 0) {
    if (info_host) *info_host = 0;
    return HKS_OK;
  }
  cudaStream_t s = as_stream(stream);
  int* dinfo = nullptr;
  Bases* db = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&dinfo), sizeof(int), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(dinfo, 0, sizeof(int), s);
  StepList sl;
  add_lu_program(sl, {LuJob{abs_ref(A), (int)n, (int)lda, abs_ref(piv), abs_ref(dinfo), kNull, kNull, 0, 0}}, false);
  if (e == cudaSuccess) e = upload_bases(make_bases(nullptr), &db, s);
  if (e == cudaSuccess) e = sl.upload(s);
  if (e == cudaSuccess) e = sl.run(db, nullptr, 0, KernelParams{}, s);
  int info = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (db) cudaFreeAsync(db, s);
  if (dinfo) cudaFreeAsync(dinfo, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_lu_factor: %s", cudaGetErrorString(e));
  if (info_host) *info_host = info;
  if (info) return set_error(HKS_ERR_SINGULAR, "singular matrix: zero pivot at elimination step %d", info - 1);
  return HKS_OK;
}

extern "C" int hks_lu_solve(const double* LU, const int32_t* piv, int64_t n, int64_t lda, double* B, int64_t ldb,
                            int64_t nrhs, void* stream) {
  if (n < 0 || lda < n || ldb < n || nrhs < 0) return set_error(HKS_ERR_INVALID, "hks_lu_solve: bad dims");
  if (n == 0 || nrhs == 0) return HKS_OK;
  cudaStream_t s = as_stream(stream);
  StepList sl;
  add_lu_solve_program(sl, {LuJob{abs_ref(LU), (int)n, (int)lda, abs_ref(piv), kNull, kNull, abs_ref(B), (int)nrhs,
                                  (int)ldb}});
  Bases* db = nullptr;
  cudaError_t e = upload_bases(make_bases(nullptr), &db, s);
  if (e == cudaSuccess) e = sl.upload(s);
  if (e == cudaSuccess) e = sl.run(db, nullptr, 0, KernelParams{}, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // before sl's device arena is freed
  if (db) cudaFreeAsync(db, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_lu_solve: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_plan_create_ex(hks_plan** out, const double* X, int64_t n, int64_t d, int64_t depth,
                                  int64_t max_rank, const int64_t* ranks_host, const hks_kernel* kern, int32_t mode) {
  if (!out || !X || !ranks_host || !kern || n < 1 || d < 1 || depth < 0 || max_rank < 1 ||
      (mode != PM_FULL && mode != PM_SUBTREE && mode != PM_TOP) || (mode == PM_TOP && depth < 1))
    return set_error(HKS_ERR_INVALID, "hks_plan_create: bad arguments");
  std::unique_ptr<hks_plan> P(new hks_plan());
  P->L = make_layout(n, depth, max_rank, mode);
  P->X = X;
  P->d = d;
  P->rank.assign(ranks_host, ranks_host + P->L.nn);
  if (!P->L.has_up(0)) P->rank[0] = 0;
  for (int64_t i = 0; i < P->L.nn; ++i) {
    if (!P->L.has_up(i)) continue;
    const int64_t cap = P->L.external(i) ? max_rank
                        : P->L.is_leaf(i) ? std::min<int64_t>(max_rank, P->L.size[i])
                                          : std::min<int64_t>(max_rank, P->R(i));
    if (P->rank[i] < 0 || P->rank[i] > cap)
      return set_error(HKS_ERR_INVALID, "hks_plan_create: rank %lld of node %lld outside [0, %lld]",
                       (long long)P->rank[i], (long long)i, (long long)cap);
  }
  P->kp = make_kernel_params(kern);
  P->kern = *kern;
  P->stack_off.assign(P->L.nn, -1);
  for (int64_t i = 0; i < P->L.first(P->L.depth); ++i) {
    P->stack_off[i] = P->stack_total;
    P->stack_total += P->R(i);
  }
  if (mode == PM_SUBTREE) {
    P->root_slot = P->stack_total;
    P->stack_total += P->rank[0];
  }
  *out = P.release();
  return HKS_OK;
}

extern "C" int hks_plan_create(hks_plan** out, const double* X, int64_t n, int64_t d, int64_t depth,
                               int64_t max_rank, const int64_t* ranks_host, const hks_kernel* kern) {
  return hks_plan_create_ex(out, X, n, d, depth, max_rank, ranks_host, kern, PM_FULL);
}

extern "C" int hks_layout_ex(int64_t n, int64_t depth, int64_t max_rank, int32_t mode, int64_t* sizes,
                             int64_t* offsets) {
  if (n < 1 || depth < 0 || depth > 40 || max_rank < 1 || mode < PM_FULL || mode > PM_TOP ||
      (mode == PM_TOP && depth < 1))
    return set_error(HKS_ERR_INVALID, "hks_layout: bad arguments n=%lld depth=%lld max_rank=%lld mode=%d",
                     (long long)n, (long long)depth, (long long)max_rank, (int)mode);
  Layout L = make_layout(n, depth, max_rank, mode);
  for (int b = 0; b < HKS_NBUF; ++b) {
    if (sizes) sizes[b] = L.total[b];
    if (offsets) std::memcpy(offsets + b * L.nn, L.off[b].data(), L.nn * sizeof(int64_t));
  }
  return HKS_OK;
}

extern "C" int hks_plan_destroy(hks_plan* P) {
  delete P;
  return HKS_OK;
}

extern "C" int hks_build_operator(hks_plan* P, void* const* buffers, void* stream) {
  if (!P || !buffers) return set_error(HKS_ERR_INVALID, "hks_build_operator: null argument");
  cudaStream_t s = as_stream(stream);
  if (P->coup_steps.empty()) {
    const Layout& L = P->L;
    std::vector<EvalDesc> ev;
    int mm = 0, mn = 0;
    for (int64_t i = 0; i < L.first(L.depth); ++i) {  // treecode.py:48-55
      const int rl = (int)P->rank[2 * i + 1], rr = (int)P->rank[2 * i + 2];
      if (rl == 0 || rr == 0) continue;
      ev.push_back(EvalDesc{make_ref(HKS_BUF_SKEL, (uint64_t)L.off[HKS_BUF_SKEL][2 * i + 1] * 8),
                            make_ref(HKS_BUF_SKEL, (uint64_t)L.off[HKS_BUF_SKEL][2 * i + 2] * 8), 0, 0, rl, rr,
                            make_ref(HKS_BUF_COUP, (uint64_t)L.off[HKS_BUF_COUP][i] * 8), rl, 0});
      mm = std::max(mm, rl);
      mn = std::max(mn, rr);
    }
    P->coup_steps.add(ST_EVAL_CM, ev, mm, mn);
    cudaError_t e = P->coup_steps.upload(s);
    if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_build_operator: %s", cudaGetErrorString(e));
  }
  cudaError_t e = run_graphed(P->coup_exec, P->coup_steps, make_bases(buffers), P->X, (int)P->d, P->kp, s, nullptr,
                              nullptr, 0, false);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_build_operator: %s", cudaGetErrorString(e));
  return HKS_OK;
}

// Evaluate and keep every leaf block K_aa (no lam) of the plan in device
// memory (treecode.py:48-51 caches them).  Must precede the first
// factorize / hmatvec of the plan (their level programs are built on first
// use and then bake the choice in).
extern "C" int hks_plan_cache_leaves(hks_plan* P, void* stream) {
  if (!P) return set_error(HKS_ERR_INVALID, "hks_plan_cache_leaves: null plan");
  if (P->leaf_cached || P->L.mode == PM_TOP) return HKS_OK;
  if (P->fact[0] || P->fact[1] || !P->mv_prog.empty() || !P->solve_prog.empty())
    return set_error(HKS_ERR_INVALID, "hks_plan_cache_leaves: the plan's programs are already built");
  const Layout& L = P->L;
  cudaStream_t s = as_stream(stream);
  P->leaf_off.assign(L.nn, -1);
  int64_t total = 0;
  int mx = 0;
  for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
    P->leaf_off[i] = total;
    total += L.size[i] * L.size[i];
    mx = std::max<int>(mx, (int)L.size[i]);
  }
  cudaError_t e = P->leaf_cache.ensure((size_t)std::max<int64_t>(total, 1) * sizeof(double));
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_plan_cache_leaves: %s", cudaGetErrorString(e));
  StepList sl;
  std::vector<EvalDesc> ev;
  for (int64_t i = L.first(L.depth); i < L.nn; ++i) {
    const int m = (int)L.size[i];
    ev.push_back(EvalDesc{kNull, kNull, L.begin[i], L.begin[i], m, m,
                          abs_ref(static_cast<double*>(P->leaf_cache.p) + P->leaf_off[i]), m, 0});
  }
  sl.add(ST_EVAL_CM, ev, mx, mx);
  e = sl.upload(s);
  Bases b{};
  Bases* db = nullptr;
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&db), sizeof(Bases), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(db, &b, sizeof(Bases), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = sl.run(db, P->X, (int)P->d, P->kp, s);
  if (db) cudaFreeAsync(db, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // the uploaded descriptors die with `sl`
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_plan_cache_leaves: %s", cudaGetErrorString(e));
  P->leaf_cached = true;
  return HKS_OK;
}

extern "C" int hks_leaf_block(hks_plan* P, int64_t leaf, double* out, void* stream) {
  if (!P || leaf < P->L.first(P->L.depth) || leaf >= P->L.nn)
    return set_error(HKS_ERR_INVALID, "hks_leaf_block: bad leaf %lld", (long long)leaf);
  const int64_t m = P->L.size[leaf];
  if (P->leaf_cached) {  // the exact values factorize / hmatvec use
    cudaError_t e = cudaMemcpyAsync(out, static_cast<const double*>(P->leaf_cache.p) + P->leaf_off[leaf],
                                    (size_t)m * m * sizeof(double), cudaMemcpyDeviceToDevice, as_stream(stream));
    if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_leaf_block: %s", cudaGetErrorString(e));
    return HKS_OK;
  }
  return hks_eval_block(P->X, P->d, &P->kern, nullptr, P->L.begin[leaf], m, nullptr, P->L.begin[leaf], m, out, m, 0,
                        0.0, stream);
}

// dgecon for every internal level on the condition stream, each level as
// soon as its LU is done (the factorization records level_ev[m] at its
// level marks); cond_done marks the last one.  Not joined back: the caller
// reads z_cond through hks_factor_stats, which waits for cond_done.
static cudaError_t launch_cond(hks_plan* P, const Bases& b) {
  cudaError_t e = cudaSuccess;
  if (!P->cond_stream) {
    if (!P->own_cond_stream) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      e = cudaStreamCreateWithPriority(&P->own_cond_stream, cudaStreamNonBlocking, lo);
      if (e != cudaSuccess) return e;
    }
    P->cond_stream = P->own_cond_stream;
  }
  if (!P->cond_done) e = cudaEventCreateWithFlags(&P->cond_done, cudaEventDisableTiming);
  if (e != cudaSuccess) return e;
  cudaStream_t cs = P->cond_stream;
  // pageable source: staged before the call returns; stream order keeps the
  // previous factorization's estimates reading their own table until done
  Bases hb = b;
  hb.p[B_VWS] = static_cast<char*>(P->cond_ws.p);  // per-matrix dlacn2 state (kGeconScratchBase)
  // through the pinned ring of a GraphCache: a pageable copy would block the
  // host until the condition stream reached it (measured: ~14 ms per call)
  static const bool htrace = getenv("HKS_HOST_TRACE") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  e = P->cond_gc.write(hb, cs);
  auto t1 = std::chrono::steady_clock::now();
  long long wt = 0, rt = 0;
  for (size_t i = 0; i < P->cond_levels.size() && e == cudaSuccess; ++i) {
    auto a = std::chrono::steady_clock::now();
    e = cudaStreamWaitEvent(cs, P->level_ev[P->cond_wait[i]], 0);
    auto b2 = std::chrono::steady_clock::now();
    if (e == cudaSuccess) e = P->cond_levels[i]->run(P->cond_gc.dev, P->X, (int)P->d, P->kp, cs);
    auto c = std::chrono::steady_clock::now();
    wt += std::chrono::duration_cast<std::chrono::microseconds>(b2 - a).count();
    rt += std::chrono::duration_cast<std::chrono::microseconds>(c - b2).count();
  }
  if (htrace)
    fprintf(stderr, "HKS_HOST cond write %lld us, waits %lld us, launches %lld us\n",
            (long long)std::chrono::duration_cast<std::chrono::microseconds>(t1 - t0).count(), wt, rt);
  if (e == cudaSuccess) e = cudaEventRecord(P->cond_done, cs);
  if (e == cudaSuccess) P->cond_pending = true;
  return e;
}

// The caller's stream hands over to the plan's high-priority stream and
// back (HKS_HIPRI=0: run on the caller's stream).
static bool hipri_enabled() {
  static const bool on = [] {
    const char* e = getenv("HKS_HIPRI");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}

static cudaError_t enter_hi(hks_plan* P, cudaStream_t s, cudaStream_t* run) {
  *run = s;
  if (!hipri_enabled()) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (!P->hi) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    e = cudaStreamCreateWithPriority(&P->hi, cudaStreamNonBlocking, hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&P->hi_in, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&P->hi_out, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  e = cudaEventRecord(P->hi_in, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(P->hi, P->hi_in, 0);
  if (e == cudaSuccess) *run = P->hi;
  return e;
}

static cudaError_t leave_hi(hks_plan* P, cudaStream_t s, cudaStream_t run) {
  if (run == s) return cudaSuccess;
  cudaError_t e = cudaEventRecord(P->hi_out, run);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, P->hi_out, 0);
  return e;
}

static int check_info(hks_plan* P, void* const* buffers, int64_t* bad_node, cudaStream_t s) {
  const Layout& L = P->L;
  std::vector<int> info(L.nn);
  const char* dinfo = static_cast<const char*>(buffers[HKS_BUF_STATS]) + L.nn * 16;
  cudaError_t e = cudaMemcpyAsync(info.data(), dinfo, L.nn * sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_factorize: %s", cudaGetErrorString(e));
  for (int64_t lev = L.depth; lev >= 0; --lev) {
    for (int64_t i = L.first(lev); i < L.first(lev) + L.count(lev); ++i) {
      if (info[i] == 0 || L.external(i)) continue;
      if (bad_node) *bad_node = i;
      if (lev == L.depth)
        return set_error(HKS_ERR_SINGULAR, "singular matrix: zero pivot at elimination step %d", info[i] - 1);
      // min |diag(Z)| of the assembled Z (solver.py:99-105): Z = I plus
      // off-diagonal blocks only (solver.py:145-147), so every diagonal
      // entry is exactly 1 -- the value is known without keeping a copy of
      // Z beside its in-place LU (a 0 x 0 Z never reaches getrf there)
      const double min_diag_z = 1.0;
      return set_error(HKS_ERR_REDUCED_SINGULAR,
                       "reduced system singular at node %lld (level %lld); smallest pivot 0 "
                       "(smallest |Z| diagonal %.3e); increase lambda or tighten tau",
                       (long long)i, (long long)lev, min_diag_z);
    }
  }
  return HKS_OK;
}

extern "C" int hks_factorize(hks_plan* P, void* const* buffers, double lam, int32_t with_cond, int64_t* bad_node,
                             void* stream) {
  if (!P || !buffers) return set_error(HKS_ERR_INVALID, "hks_factorize: null argument");
  if (!(lam >= 0.0)) return set_error(HKS_ERR_INVALID, "lambda must be nonnegative");
  cudaStream_t s = as_stream(stream);
  const int which = with_cond ? 1 : 0;
  if (!P->fact[which]) {
    P->fact[which].reset(new StepList());
    if (which == 1) {
      P->cond_levels.clear();
      P->cond_wait.clear();
    }
    build_factorize(*P, with_cond != 0, *P->fact[which], which == 1 ? &P->cond_levels : nullptr,
                    which == 1 ? &P->cond_wait : nullptr);
    cudaError_t e = P->fact[which]->upload(s);
    for (auto& c : P->cond_levels)
      if (e == cudaSuccess && which == 1) e = c->upload(s);
    if (e == cudaSuccess) e = P->fws.ensure(std::max<size_t>(factorize_workspace(*P), 1) * sizeof(double));
    if (e == cudaSuccess && which == 1)
      e = P->cond_ws.ensure(std::max<size_t>(cond_scratch_elems(*P), 1) * sizeof(double));
    if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_factorize: %s", cudaGetErrorString(e));
  }
  Bases b = make_bases(buffers);
  b.p[B_FWS] = static_cast<char*>(P->fws.p);
  b.lam = lam;
  const size_t nev = P->fact[which]->marks().size() + 1;
  while (P->level_ev.size() < nev) {
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    P->level_ev.push_back(ev);
  }
  static const bool htrace = getenv("HKS_HOST_TRACE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t0 = now();
  cudaStream_t rs = s;
  cudaError_t e = enter_hi(P, s, &rs);
  if (e == cudaSuccess)
    e = run_graphed(P->fact_graphs[which], *P->fact[which], b, P->X, (int)P->d, P->kp, rs, P->level_ev.data(),
                    buffers[HKS_BUF_STATS], P->L.nn * 3 * sizeof(double));
  const auto t1 = now();
  if (e == cudaSuccess) e = leave_hi(P, s, rs);
  if (e == cudaSuccess && which == 1 && !P->cond_levels.empty()) e = launch_cond(P, b);
  const auto t2 = now();
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_factorize: %s", cudaGetErrorString(e));
  if (bad_node) *bad_node = -1;
  const int rc = check_info(P, buffers, bad_node, s);
  if (htrace) {
    const auto t3 = now();
    auto us = [](std::chrono::steady_clock::duration d) {
      return (long long)std::chrono::duration_cast<std::chrono::microseconds>(d).count();
    };
    fprintf(stderr, "HKS_HOST factorize launch %lld us, cond %lld us, sync %lld us\n", us(t1 - t0), us(t2 - t1),
            us(t3 - t2));
  }
  return rc;
}

extern "C" int hks_factor_stats(hks_plan* P, void* const* buffers, double* z_cond, int32_t* info, void* stream) {
  if (!P || !buffers) return set_error(HKS_ERR_INVALID, "hks_factor_stats: null argument");
  cudaStream_t s = as_stream(stream);
  const Layout& L = P->L;
  if (P->cond_pending) {  // the dgecon estimates run on the condition stream
    cudaError_t e = cudaEventSynchronize(P->cond_done);
    if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_factor_stats: %s", cudaGetErrorString(e));
  }
  std::vector<double> st(3 * L.nn);
  cudaError_t e = cudaMemcpyAsync(st.data(), buffers[HKS_BUF_STATS], st.size() * sizeof(double),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_factor_stats: %s", cudaGetErrorString(e));
  const int* inf = reinterpret_cast<const int*>(st.data() + 2 * L.nn);
  for (int64_t i = 0; i < L.nn; ++i) {
    if (info) info[i] = inf[i];
    if (!z_cond) continue;
    if (L.is_leaf(i)) {
      z_cond[i] = 0.0;
    } else {  // solver.py:106-107: cond = 1 / rcond, inf when rcond == 0
      const double rc = st[L.nn + i];
      z_cond[i] = rc > 0 ? 1.0 / rc : std::numeric_limits<double>::infinity();
    }
  }
  return HKS_OK;
}

// Stream the dgecon estimates run on (default: an internal lowest-priority
// stream).  A caller that owns the factor storage's allocator passes its
// own stream so it can mark the storage in use there.
extern "C" int hks_set_cond_stream(hks_plan* P, void* stream) {
  if (!P) return set_error(HKS_ERR_INVALID, "hks_set_cond_stream: null plan");
  if (P->cond_pending && P->cond_done) cudaEventSynchronize(P->cond_done);
  P->cond_stream = stream ? as_stream(stream) : P->own_cond_stream;
  return HKS_OK;
}

// `stream` waits (device-side) for the last factorization's dgecon estimates.
extern "C" int hks_cond_wait(hks_plan* P, void* stream) {
  if (!P) return set_error(HKS_ERR_INVALID, "hks_cond_wait: null plan");
  if (!P->cond_pending) return HKS_OK;
  const cudaError_t e = cudaStreamWaitEvent(as_stream(stream), P->cond_done, 0);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_cond_wait: %s", cudaGetErrorString(e));
  return HKS_OK;
}

static VecProgram* get_prog(std::map<int64_t, std::unique_ptr<VecProgram>>& m, int64_t k) {
  auto it = m.find(k);
  if (it != m.end()) return it->second.get();
  VecProgram* v = new VecProgram();
  m[k].reset(v);
  return v;
}

// One program half (part 0 whole, 1 up, 2 down; see build_solve) with its
// own graph; both halves of a subtree plan share the workspace.
static cudaError_t run_vec_part(hks_plan* P, VecProgram* v, int part, Bases& bb, const void* xin, void* xout,
                                cudaStream_t s) {
  bb.p[B_VWS] = (char*)v->ws.p;
  bb.p[B_XIN] = (char*)xin;
  bb.p[B_XOUT] = (char*)xout;
  StepList& sl = part == 2 ? v->down : v->steps;
  GraphCache& gc = part == 2 ? v->down_graphs : v->graphs;
  cudaStream_t rs = s;
  cudaError_t e = enter_hi(P, s, &rs);
  if (e == cudaSuccess) e = run_graphed(gc, sl, bb, P->X, (int)P->d, P->kp, rs, nullptr, nullptr, 0);
  if (e == cudaSuccess) e = leave_hi(P, s, rs);
  return e;
}

static int check_part(hks_plan* P, int part, const void* xchg, const char* who) {
  const bool sub = P->L.mode == PM_SUBTREE;
  if (part < 0 || part > 2 || (sub && part == 0) || (!sub && part != 0))
    return set_error(HKS_ERR_INVALID, "%s: part %d does not fit a mode-%d plan", who, part, P->L.mode);
  if (sub && !xchg && P->rank[0] > 0) return set_error(HKS_ERR_INVALID, "%s: subtree plans need the exchange block", who);
  return HKS_OK;
}

extern "C" int hks_solve_part(hks_plan* P, void* const* buffers, const double* b, double* x, int64_t k, int32_t part,
                              double* xchg, void* stream) {
  if (!P || !buffers || !b || !x || k < 0) return set_error(HKS_ERR_INVALID, "hks_solve: bad arguments");
  if (int rc = check_part(P, part, xchg, "hks_solve")) return rc;
  if (k == 0) return HKS_OK;
  cudaStream_t s = as_stream(stream);
  VecProgram* v = get_prog(P->solve_prog, k);
  if (v->steps.empty() && v->down.empty()) {
    const bool sub = P->L.mode == PM_SUBTREE;
    build_solve(*P, k, sub ? 1 : 0, v->steps);
    if (sub) build_solve(*P, k, 2, v->down);
    cudaError_t e = v->steps.upload(s);
    if (e == cudaSuccess) e = v->down.upload(s);
    if (e == cudaSuccess) e = v->ws.ensure(std::max<size_t>(3 * P->stack_total * k, 1) * sizeof(double));
    if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_solve: %s", cudaGetErrorString(e));
  }
  Bases bb = make_bases(buffers);
  bb.p[B_VIN] = (char*)b;
  bb.p[B_VOUT] = (char*)x;
  cudaError_t e = run_vec_part(P, v, part, bb, xchg, xchg, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_solve: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_solve(hks_plan* P, void* const* buffers, const double* b, double* x, int64_t k, void* stream) {
  return hks_solve_part(P, buffers, b, x, k, 0, nullptr, stream);
}

extern "C" int hks_hmatvec_part(hks_plan* P, void* const* buffers, const double* w, double* u, int64_t k, double lam,
                                int32_t part, double* xchg, void* stream) {
  if (!P || !buffers || !w || !u || k < 0 || w == u) return set_error(HKS_ERR_INVALID, "hks_hmatvec: bad arguments");
  if (int rc = check_part(P, part, xchg, "hks_hmatvec")) return rc;
  if (k == 0) return HKS_OK;
  cudaStream_t s = as_stream(stream);
  VecProgram* v = get_prog(P->mv_prog, k);
  if (v->steps.empty() && v->down.empty()) {
    const bool sub = P->L.mode == PM_SUBTREE;
    build_matvec(*P, k, sub ? 1 : 0, v->steps);
    if (sub) build_matvec(*P, k, 2, v->down);
    cudaError_t e = v->steps.upload(s);
    if (e == cudaSuccess) e = v->down.upload(s);
    if (e == cudaSuccess) e = v->ws.ensure(std::max<size_t>(2 * P->stack_total * k, 1) * sizeof(double));
    if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_hmatvec: %s", cudaGetErrorString(e));
  }
  Bases bb = make_bases(buffers);
  bb.p[B_VIN] = (char*)w;
  bb.p[B_VOUT] = (char*)u;
  bb.lam = lam;
  cudaError_t e = run_vec_part(P, v, part, bb, xchg, xchg, s);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_hmatvec: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_hmatvec(hks_plan* P, void* const* buffers, const double* w, double* u, int64_t k, double lam,
                           void* stream) {
  return hks_hmatvec_part(P, buffers, w, u, k, lam, 0, nullptr, stream);
}

extern "C" int hks_upward_offsets(hks_plan* P, int64_t k, int64_t* offsets, int64_t* lds, int64_t* total) {
  if (!P) return set_error(HKS_ERR_INVALID, "null plan");
  if (offsets) offsets[0] = -1;
  if (lds) lds[0] = 0;
  for (int64_t i = 1; i < P->L.nn; ++i) {
    const int64_t p = (i - 1) / 2;
    const int64_t row = (i == 2 * p + 1) ? 0 : P->rank[2 * p + 1];
    if (offsets) offsets[i] = P->stack_off[p] * k + row;
    if (lds) lds[i] = P->R(p);
  }
  if (total) *total = P->stack_total * k;
  return HKS_OK;
}

extern "C" int hks_upward(hks_plan* P, void* const* buffers, const double* w, int64_t k, double* out, void* stream) {
  if (!P || !buffers || !w || !out || k < 1) return set_error(HKS_ERR_INVALID, "hks_upward: bad arguments");
  cudaStream_t s = as_stream(stream);
  VecProgram* v = get_prog(P->up_prog, k);
  if (v->steps.empty() && P->L.depth > 0) {
    build_upward(*P, k, 0, v->steps);
    cudaError_t e = v->steps.upload(s);
    if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_upward: %s", cudaGetErrorString(e));
  }
  Bases bb = make_bases(buffers);
  bb.p[B_VIN] = (char*)w;
  bb.p[B_VWS] = (char*)out;  // stacked slots written straight into the caller's buffer
  cudaError_t e = run_graphed(v->graphs, v->steps, bb, P->X, (int)P->d, P->kp, s, nullptr, nullptr, 0, false);
  if (e != cudaSuccess) return set_error(HKS_ERR_CUDA, "hks_upward: %s", cudaGetErrorString(e));
  return HKS_OK;
}

extern "C" int hks_profile(int32_t enable, double* out_host) {
  // enable: 1 start (reset), 0 stop; out_host[kind * 4 + {launches, ms, flops, bytes}]
  // for the kNumKinds step kinds (GEMM, COPY, GETRF, GETRS, GECON, EVAL_CM, EVAL_RM, KSUM).
  cudaDeviceSynchronize();
  for (auto& p : g_prof.pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    if (getenv("HKS_TRACE")) fprintf(stderr, "HKS_TRACE %d %.5f %.6g %.6g\n", p.kind, ms, p.flops, p.bytes);
    g_prof.launches[p.kind] += 1;
    g_prof.ms[p.kind] += ms;
    g_prof.flops[p.kind] += p.flops;
    g_prof.bytes[p.kind] += p.bytes;
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  g_prof.pending.clear();
  if (out_host)
    for (int k = 0; k < kNumKinds; ++k) {
      out_host[4 * k + 0] = g_prof.launches[k];
      out_host[4 * k + 1] = g_prof.ms[k];
      out_host[4 * k + 2] = g_prof.flops[k];
      out_host[4 * k + 3] = g_prof.bytes[k];
    }
  if (enable) {
    for (int k = 0; k < kNumKinds; ++k) g_prof.launches[k] = g_prof.ms[k] = g_prof.flops[k] = g_prof.bytes[k] = 0;
  }
  g_prof.on = enable != 0;
  return HKS_OK;
}

extern "C" long long hks_launch_count(void) { return g_launches; }

// Device milliseconds of each level of the last hks_factorize on this plan:
// ms_host[level] for level = 0..depth (the leaf level is `depth`).
extern "C" int hks_factor_level_ms(hks_plan* P, double* ms_host) {
  if (!P || !ms_host) return set_error(HKS_ERR_INVALID, "hks_factor_level_ms: null argument");
  const int64_t nl = P->L.depth + 1;
  if ((int64_t)P->level_ev.size() < nl + 1) return set_error(HKS_ERR_INVALID, "hks_factor_level_ms: not factorized");
  cudaEventSynchronize(P->level_ev[nl]);
  for (int64_t m = 0; m < nl; ++m) {  // mark m: leaf level first, then depth-1 .. 0
    float ms = 0.f;
    cudaEventElapsedTime(&ms, P->level_ev[m], P->level_ev[m + 1]);
    const int64_t level = P->L.depth - m;
    ms_host[level] = ms;
  }
  return HKS_OK;
}
