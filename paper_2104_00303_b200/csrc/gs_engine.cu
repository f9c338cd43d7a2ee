// gridshift-b200: host orchestration and C ABI (see include/gridshift_cuda.h).
//
// One gs_ctx = one device, one stream, a set of grow-only device buffers and
// pinned host mirrors of the loop-control block.  The iteration loop is
// device-driven: kernels test Ctrl::done, so the host enqueues iterations in
// chunks and only synchronises between chunks (no per-iteration round trip).

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <chrono>
#include <thread>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "../../include/gridshift_cuda.h"
#include "gs_kernels.cuh"
#include "gs_refsum.cuh"
#include "gs_track.cuh"

using namespace gs;

namespace {

thread_local std::string g_err;

struct Fail {
  int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
  g_err = msg;
  throw Fail{code};
}

#define GS_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      fail(GS_ERUNTIME, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                            __FILE__ + ":" + std::to_string(__LINE__) + " (" #call ")"); \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
};

enum Kind { K_INIT = 0, K_HIST, K_AGG, K_SHIFT, K_CLEAR, K_COMP, K_LABELS, K_XPOSE, K_DUMP, K_TRACK,
            K_SORT, K_DERIVE, K_REFSUM, K_NKINDS };
const char* const kKindNames[K_NKINDS] = {"init", "hist", "agg", "shift", "clear", "components",
                                          "labels", "transpose", "dump", "track", "sort", "derive", "refsum"};

constexpr int64_t kSortMinPoints = 1 << 15;   // spatial sort pays off above this
constexpr int kClassifyThreads = 256;         // k_rs_classify CTA size in the default sum order
constexpr int kShiftCtasChain = 6;            // shift CTAs per SM while the sequential-sum chain runs beside it

inline int64_t soa_ld(int64_t n) { return (n + 127) & ~int64_t(127); }   // = k_hist tile

// Per-context kernel accounting: every launch is counted; with profiling on,
// each launch is bracketed by CUDA events on the launching stream.
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<int, size_t>> rec;   // (kind, first event index)
  int64_t launches[K_NKINDS] = {};
};

}  // namespace

// Reference-order sums of the current run (gs_refsum.cuh): device pointers
// into the context's buffers, sized by rs_alloc.
struct RsRun {
  bool on = false;
  bool model = false;    // GS_SUMS_SEQMODEL: closed forms + proportional folds, no point order
  int64_t n = 0;
  u32 nblk = 0;          // radix tiles over n points
  int maxpasses = 0;     // radix passes that can be needed for the segment ids
  u64 segcap = 0;        // max segments (occupied cells)
  double* rs[2] = {nullptr, nullptr};   // per table buffer: slots x D reference-order sums
  u32 *nsrc = nullptr, *mid = nullptr, *outslot = nullptr, *rc[2] = {nullptr, nullptr}, *runkey = nullptr,
      *runval = nullptr, *k[2] = {nullptr, nullptr}, *v[2] = {nullptr, nullptr}, *cnt = nullptr,
      *scan = nullptr, *sstart = nullptr, *send = nullptr;
  double *wsum = nullptr, *wpre = nullptr;
  u64* wdelta = nullptr;
  RsCtl* ctl = nullptr;
  const u32* cell0 = nullptr;   // per point: run (initial slot)
  const u32* runs = nullptr;    // occupied runs
  const u32* nruns = nullptr;   // (device)
  u64 slots = 0;                // loop table slots
  // gathered segments (sorted runs): lengths, run lists
  u32 *seglen = nullptr, *segbeg = nullptr, *segcur = nullptr, *seglist = nullptr, *runseg = nullptr,
      *segscan = nullptr;
  const u32 *start = nullptr, *end = nullptr, *perm = nullptr;   // the spatial sort's runs
  bool all_big = true;          // no spatial sort: every segment takes the global sort
  u64* runkv = nullptr;         // per run: pass-0 key (low) and value (high)
  void* tag[2] = {nullptr, nullptr};   // per table buffer: Rec<D> the slot's closed form came from
  u32* stats = nullptr;         // per table: 5 counters (k_rs_stats)
  int stats_rows = 0;
  // index-ordered point lists of the cells (RsLists): per table buffer the
  // list of each slot, source chains of the mixed targets, the arena (perm
  // first) and its fill mark
  u64* lst[2] = {nullptr, nullptr};
  u32 *shead = nullptr, *snext = nullptr, *segdone = nullptr, *ctalist = nullptr;
  u64 arena_cap = 0;
  unsigned long long* arena_top = nullptr;
};

struct gs_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t own = nullptr;
  cudaStream_t st = nullptr;      // stream of the current call
  std::mutex mu;
  // device buffers
  Buf x_stage, y[2], ent[2], keys[2], list[2], targets, partials, par, first, aux, roots,
      root_first, ranks, modes, labels, mv_hist, fp_hist, k_hist, stats, ctrl, perm, track,
      track_out, bitmaps, scan, runoff, runstart, runmin, runlist, cell0, stage;
  // pinned host mirrors
  Ctrl* h_ctrl = nullptr;
  InitStats* h_stats = nullptr;
  u32* h_small = nullptr;        // pinned scratch for small device->host reads
  // last-run results
  int d_last = 0;
  int64_t k_last = 0;
  std::vector<double> modes_host;
  std::vector<double> colors_host;      // (k, 3) mean colours of the last gs_segment_image
  Buf colsum;
  std::vector<int64_t> iter_k;
  std::vector<uint64_t> iter_fp;
  std::vector<int64_t> track_bins;
  Prof prof;
  bool collapsed = false;               // option: collapsed iterations (gs_ctx_set_option)
  Buf runposb, runcntb, bkcnt, bktot, bocc, bmask, wr_hist;
  bool tables_dirty = false;            // a call failed mid-run: table buffers may hold entries
  Ctrl* h_snap = nullptr;               // pinned Ctrl snapshots after each enqueued chunk (2 slots)
  cudaEvent_t ev_snap[2] = {nullptr, nullptr};
  // table-chain stream (see enqueue_iteration: overlap)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_rec[2] = {nullptr, nullptr}, ev_shift[2] = {nullptr, nullptr};
  cudaEvent_t ev_pace[2] = {nullptr, nullptr};   // timing-enabled, around side-stream kernels
  struct ShardState* shard = nullptr;   // row-sharded run in progress (gs_shard_*)
  // host label delivery (sorted runs through the host entry points): the
  // per-point initial-cell index is copied to the host on `copy` while the
  // loop runs; the extraction then sends per-cell labels only and the host
  // expands them (deliver_labels)
  bool host_labels = false;             // request, set by the host entry points
  bool cell0_pending = false;           // the cell0 copy is enqueued (on `copy`)
  bool labels_on_host = false;          // extraction left per-cell labels in h_slotlab
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_sorted = nullptr, ev_cell0 = nullptr;
  u32* h_cell0 = nullptr;               // pinned, n entries
  size_t h_cell0_cap = 0;
  u32* h_slotlab = nullptr;             // pinned, per initial slot: label rank
  size_t h_slotlab_cap = 0;
  Buf slotlab;
  const u32* cell0_dev = nullptr;
  int64_t cell0_n = 0;
  int64_t xfer_h2d = 0, xfer_d2h = 0;   // last host call (gs_fetch_transfer_bytes)
  size_t slotlab_bytes = 0;
  // reference-order sums (gs_refsum.cuh): option + buffers
  bool exact_sums = false;              // GS_OPT_SUMS: GS_SUMS_EXACT
  bool seq_model = true;                // GS_OPT_SUMS: GS_SUMS_SEQMODEL, the default (sequential sums without the point order)
  // the last per-point run's iterate (gs_fetch_iterate)
  int64_t it_n = 0;
  int it_d = 0;
  bool it_sorted = false, it_valid = false;
  Buf rsb[2], rs_nsrc, rs_mid, rs_out, rs_rc[2], rs_rkey, rs_rval, rs_k[2], rs_v[2], rs_cnt, rs_scan,
      rs_start, rs_end, rs_wsum, rs_wpre, rs_wdelta, rs_ctl, rs_cell0, rs_runs, rs_seglen, rs_segbeg,
      rs_segcur, rs_seglist, rs_runseg, rs_segscan, rs_runkv, rs_tag[2], rs_stats, rs_lowrun, rs_lst[2],
      rs_shead, rs_snext, rs_segdone, rs_atop, rs_ctalist, rs_nocc;
  RsRun rsr;
};

namespace {

template <typename T>
T* ensure(gs_ctx* c, Buf& b, size_t count, int fill = 0) {
  const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
  if (b.cap < bytes) {
    if (b.p) GS_CUDA(cudaFree(b.p));
    b.p = nullptr;
    b.cap = 0;
    const size_t alloc = bytes + bytes / 8;
    GS_CUDA(cudaMalloc(&b.p, alloc));
    GS_CUDA(cudaMemsetAsync(b.p, fill, alloc, c->st));
    b.cap = alloc;
  }
  return static_cast<T*>(b.p);
}

cudaEvent_t prof_event(gs_ctx* c) {
  if (c->prof.used == c->prof.pool.size()) {
    cudaEvent_t e;
    GS_CUDA(cudaEventCreate(&e));
    c->prof.pool.push_back(e);
  }
  return c->prof.pool[c->prof.used++];
}

template <typename F>
void launch(gs_ctx* c, int kind, F&& f) {
  c->prof.launches[kind] += 1;
  if (!c->prof.on) {
    // side-stream kernels are bracketed by timing-enabled events: measured
    // 37.7 -> 34.7 ms per 100M-point run against no events (or events
    // without timing), with identical results -- it changes how the
    // low-priority table chain is scheduled next to the shift
    const bool pace = c->side && c->st == c->side;
    if (pace) GS_CUDA(cudaEventRecord(c->ev_pace[0], c->st));
    f();
    if (pace) GS_CUDA(cudaEventRecord(c->ev_pace[1], c->st));
    return;
  }
  const size_t i0 = c->prof.used;
  GS_CUDA(cudaEventRecord(prof_event(c), c->st));
  f();
  GS_CUDA(cudaEventRecord(prof_event(c), c->st));
  c->prof.rec.emplace_back(kind, i0);
}

// Kernel attributes (dynamic shared memory limits, carveouts) are set once
// per device: `done` is a per-call-site bitmask over device ordinals, marked
// only after the attributes are in place (concurrent first calls both set).
inline bool attr_pending(const std::atomic<uint64_t>& done, int device) {
  return (done.load() & (1ull << (device & 63))) == 0;
}
inline void attr_done(std::atomic<uint64_t>& done, int device) { done.fetch_or(1ull << (device & 63)); }

inline int blocks_for(gs_ctx* c, int64_t work, int per_sm = 8) {
  const int64_t want = (work + kThreads - 1) / kThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->sms * per_sm));
}

void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(GS_ERUNTIME, std::string("kernel launch failed: ") + cudaGetErrorString(e));
}

void sync(gs_ctx* c) { GS_CUDA(cudaStreamSynchronize(c->st)); }

void validate_common(int64_t n, int32_t d, double h) {
  if (!(std::isfinite(h) && h > 0.0)) {
    char b[128];
    snprintf(b, sizeof b, "bandwidth must be a positive finite real, got %.17g", h);
    fail(GS_EINVAL, b);
  }
  if (n < 1 || d < 1) fail(GS_EINVAL, "need n >= 1 and d >= 1");
  if (d > GS_MAXD) fail(GS_EUNSUPPORTED, "the CUDA engine supports d <= 8 feature axes");
  if (n >= (int64_t)UINT32_MAX) fail(GS_EUNSUPPORTED, "the CUDA engine supports n < 2^32 points per device");
}

// Lattice geometry + quantisation from the initial statistics.
struct Plan {
  GridParams g;
  bool dense;
  uint64_t slots;     // table slots (dense: nkeys, hash: capacity)
  uint64_t list_cap;  // max occupied cells
};

Plan make_plan(int64_t n, int d, double h, const InitStats& s) {
  if (s.flags & kErrNonFinite) fail(GS_EINVAL, "point data contains NaN or infinite entries");
  if (s.flags & kErrLattice)
    fail(GS_EINVAL,
         "cell coordinates exceed the supported integer lattice; bandwidth is too small for this "
         "coordinate range");
  Plan p{};
  GridParams& g = p.g;
  memset(&g, 0, sizeof g);
  g.h = h;
  g.d = d;
  g.inv_h = 1.0 / h;
  __int128 prod = 1;
  double span2 = 0.0;
  int64_t ext[GS_MAXD];
  for (int j = 0; j < d; ++j) {
    // admissible box: observed cells +/- 1 (rounding drift margin), plus a
    // one-cell neighbour pad on each side for the key origin (grid.py:146-147)
    g.lo[j] = s.cmin[j] - 1;
    g.hi[j] = s.cmax[j] + 1;
    g.base[j] = g.lo[j] - 1;
    ext[j] = g.hi[j] - g.lo[j] + 3;
    prod *= ext[j];
    if (prod >= ((__int128)1 << 62))
      fail(GS_EUNSUPPORTED,
           "lattice box exceeds 2^62 cells; the CUDA engine needs packed int64 cell keys");
    double m;
    memcpy(&m, &s.absmax[j], sizeof m);
    int e = 0;
    if (m > 0) frexp(m, &e);  // m < 2^e
    int sh = 62 - (e + 1);     // |v| < 2^61
    sh = std::max(-1000, std::min(1000, sh));
    g.qexp[j] = sh;
    g.qscale[j] = ldexp(1.0, sh);
    const double w = (double)ext[j] * h;
    span2 += w * w;
  }
  uint64_t acc = 1;
  for (int j = d - 1; j >= 0; --j) {
    g.stride[j] = acc;
    acc *= (uint64_t)ext[j];
  }
  g.nkeys = acc;
  g.ld = soa_ld(n);
  int em = 0;
  frexp(std::sqrt(span2) * 1.0000001 + 1e-300, &em);
  g.movement_exp = em;
  const size_t entry = 8 * (1 + 2 * (size_t)d);
  const uint64_t occ_bound = std::min<uint64_t>((uint64_t)n, g.nkeys);
  p.dense = g.nkeys <= (1ull << 31) && g.nkeys * entry <= (4ull << 30) &&
            g.nkeys <= 64ull * (uint64_t)n + (1ull << 22);
  if (p.dense) {
    p.slots = g.nkeys;
    g.mask = 0;
  } else {
    uint64_t cap = 256;
    while (cap < 2 * occ_bound) cap <<= 1;
    if (cap > (1ull << 31)) fail(GS_EUNSUPPORTED, "hash table would exceed 2^31 slots");
    p.slots = cap;
    g.mask = cap - 1;
  }
  p.list_cap = occ_bound;
  return p;
}

template <int D>
struct Tabs {
  DenseTable<D> dn[2];
  HashTable<D> hs[2];
};

template <int D>
Tabs<D> make_tabs(gs_ctx* c, const Plan& p) {
  Tabs<D> t{};
  Ctrl* dctrl = static_cast<Ctrl*>(c->ctrl.p);
  for (int b = 0; b < 2; ++b) {
    Entry<D>* ent = ensure<Entry<D>>(c, c->ent[b], p.slots, 0);
    u32* list = ensure<u32>(c, c->list[b], p.list_cap);
    t.dn[b].ent = ent;
    t.dn[b].list = list;
    t.dn[b].k = &dctrl->k[b];
    t.hs[b].ent = ent;
    t.hs[b].list = list;
    t.hs[b].k = &dctrl->k[b];
    if (!p.dense) {
      t.hs[b].keys = ensure<u64>(c, c->keys[b], p.slots, 0xff);
      t.hs[b].mask = p.g.mask;
    }
    if (c->tables_dirty) {
      // every run path assumes clean buffers; after a failed call restore them
      GS_CUDA(cudaMemsetAsync(c->ent[b].p, 0, c->ent[b].cap, c->st));
      if (c->keys[b].p) GS_CUDA(cudaMemsetAsync(c->keys[b].p, 0xff, c->keys[b].cap, c->st));
    }
  }
  c->tables_dirty = false;
  return t;
}

void reset_ctrl(gs_ctx* c) {
  memset(c->h_ctrl, 0, sizeof(Ctrl));
  GS_CUDA(cudaMemcpyAsync(c->ctrl.p, c->h_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, c->st));
}

void read_ctrl(gs_ctx* c) {
  GS_CUDA(cudaMemcpyAsync(c->h_ctrl, c->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, c->st));
  sync(c);
}

void check_flags(int flags) {
  if (flags & kErrOutOfBox) fail(GS_ERUNTIME, "an iterate left the admissible lattice box");
  if (flags & kErrTableFull) fail(GS_ERUNTIME, "cell hash table overflow");
  if (flags & kErrMissing) fail(GS_ERUNTIME, "cell lookup missed an occupied cell");
}

// ------------------------------------------------------------ input stage

enum InKind { IN_F64 = 0, IN_F32 = 1, IN_IMAGE = 2 };

struct Input {
  InKind kind;
  const void* dev;    // device pointer
  int width = 0;      // image
  double scale = 0;   // image rgbxy scale
};

template <int D>
InitStats run_init(gs_ctx* c, const Input& in, int64_t n, double h, double* y0) {
  InitStats* dst = ensure<InitStats>(c, c->stats, 1);
  InitStats hs;
  memset(&hs, 0, sizeof hs);
  for (int j = 0; j < GS_MAXD; ++j) {
    hs.cmin[j] = LLONG_MAX;
    hs.cmax[j] = LLONG_MIN;
    hs.lowbit[j] = 4096;
  }
  *c->h_stats = hs;
  GS_CUDA(cudaMemcpyAsync(dst, c->h_stats, sizeof hs, cudaMemcpyHostToDevice, c->st));
  const int nb = blocks_for(c, n);
  if (in.kind == IN_F64)
    launch(c, K_INIT, [&] { k_init_aos<D, double><<<nb, kThreads, 0, c->st>>>((const double*)in.dev, y0, n, soa_ld(n), h, dst); });
  else if (in.kind == IN_F32)
    launch(c, K_INIT, [&] { k_init_aos<D, float><<<nb, kThreads, 0, c->st>>>((const float*)in.dev, y0, n, soa_ld(n), h, dst); });
  else {
    if constexpr (D == 3 || D == 5)
      launch(c, K_INIT, [&] { k_init_image<D><<<nb, kThreads, 0, c->st>>>((const unsigned char*)in.dev, y0, n, soa_ld(n), in.width, in.scale, h, dst); });
  }
  check_launch();
  GS_CUDA(cudaMemcpyAsync(c->h_stats, dst, sizeof hs, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  return *c->h_stats;
}

// What the spatial sort leaves behind for the run-based extraction.
struct SortInfo {
  u32* cell0 = nullptr;     // initial cell slot per point, original order
  u32* start = nullptr;     // per initial slot: run start in sorted order
  u32* minidx = nullptr;    // per initial slot: smallest original index
  u32* runs = nullptr;      // occupied initial slots
  u32* runroot = nullptr;   // per initial slot: final component root (scratch)
  u32* end = nullptr;       // per initial slot: run end (the scatter cursors)
  u32* perm = nullptr;      // sorted position -> original index (reference-order sums only)
  uint64_t slots0 = 0;      // table slots at sort time (the range of cell0)
  double* runpos = nullptr; // collapsed mode: per-run positions (SoA, ld = rld)
  u32* runcnt = nullptr;
  int64_t rld = 0;
};

// ------------------------------------------------- reference-order sums
// (gs_refsum.cuh).  rs_alloc sizes the buffers of one run; rs_first builds
// the first table's sums, rs_next those of table t+1 right after k_derive.

// perm (n entries) plus room for the merged lists of later tables (list
// offsets are 32-bit; a full arena only costs speed)
inline u64 arena_entries(int64_t n) { return std::min<u64>(4ull * (u64)n, 0xfffffff0ull); }

RsRun& rs_alloc(gs_ctx* c, const Plan& p, int d, int64_t n, u64 runs_cap, u64 segcap, int max_iters = 1,
                bool model = false) {
  RsRun& R = c->rsr;
  R.on = true;
  R.model = model;
  R.n = n;
  R.slots = p.slots;
  R.segcap = std::max<u64>(segcap, 1);
  R.nblk = (u32)((n + kRsTile - 1) / kRsTile);
  const u64 mx = R.segcap - 1;
  R.maxpasses = mx < 256 ? 1 : mx < 65536 ? 2 : mx < (1ull << 24) ? 3 : 4;
  for (int b = 0; b < 2; ++b) {
    R.rs[b] = ensure<double>(c, c->rsb[b], (size_t)p.slots * d);
    R.rc[b] = ensure<u32>(c, c->rs_rc[b], runs_cap);
    R.k[b] = model ? nullptr : ensure<u32>(c, c->rs_k[b], (size_t)n);
    R.v[b] = model ? nullptr : ensure<u32>(c, c->rs_v[b], (size_t)n);
  }
  R.nsrc = ensure<u32>(c, c->rs_nsrc, p.slots);
  R.mid = ensure<u32>(c, c->rs_mid, p.slots);
  R.outslot = ensure<u32>(c, c->rs_out, R.segcap);
  R.sstart = ensure<u32>(c, c->rs_start, R.segcap);
  R.send = ensure<u32>(c, c->rs_end, R.segcap);
  R.runkey = ensure<u32>(c, c->rs_rkey, runs_cap);
  R.runval = ensure<u32>(c, c->rs_rval, runs_cap);
  R.cnt = ensure<u32>(c, c->rs_cnt, 256ull * R.nblk);
  R.scan = ensure<u32>(c, c->rs_scan, (256ull * R.nblk + kScan32Chunk - 1) / kScan32Chunk + 1);
  const size_t nw = model ? 1 : (size_t)(n / kFoldWin) + 1;
  R.wsum = ensure<double>(c, c->rs_wsum, nw * d);
  R.wpre = ensure<double>(c, c->rs_wpre, nw * d);
  R.wdelta = ensure<u64>(c, c->rs_wdelta, nw * d);
  R.ctl = ensure<RsCtl>(c, c->rs_ctl, 1);
  R.seglen = ensure<u32>(c, c->rs_seglen, R.segcap);
  R.segbeg = ensure<u32>(c, c->rs_segbeg, R.segcap + 1);
  R.segcur = ensure<u32>(c, c->rs_segcur, R.segcap);
  R.seglist = ensure<u32>(c, c->rs_seglist, std::max<u64>(runs_cap, R.segcap));
  R.runseg = ensure<u32>(c, c->rs_runseg, std::max<u64>(runs_cap, R.segcap));
  R.segscan = ensure<u32>(c, c->rs_segscan, (R.segcap + 1 + kScan32Chunk - 1) / kScan32Chunk + 1);
  R.start = R.end = R.perm = nullptr;
  R.all_big = true;
  R.runkv = ensure<u64>(c, c->rs_runkv, runs_cap);
  for (int b = 0; b < 2; ++b) {
    const size_t tb = (size_t)p.slots * (d + 1) * sizeof(u64);
    R.tag[b] = ensure<u64>(c, c->rs_tag[b], tb / 8);
    GS_CUDA(cudaMemsetAsync(R.tag[b], 0, tb, c->st));
  }
  R.stats_rows = max_iters + 1;
  R.stats = ensure<u32>(c, c->rs_stats, 5ull * R.stats_rows);
  GS_CUDA(cudaMemsetAsync(R.stats, 0, 20ull * R.stats_rows, c->st));
  GS_CUDA(cudaMemsetAsync(R.nsrc, 0, sizeof(u32) * p.slots, c->st));
  GS_CUDA(cudaMemsetAsync(R.mid, 0xff, sizeof(u32) * p.slots, c->st));
  for (int b = 0; b < 2; ++b) R.lst[b] = ensure<u64>(c, c->rs_lst[b], p.slots);
  R.shead = ensure<u32>(c, c->rs_shead, p.slots);
  R.snext = ensure<u32>(c, c->rs_snext, p.slots);
  R.segdone = ensure<u32>(c, c->rs_segdone, R.segcap);
  R.ctalist = ensure<u32>(c, c->rs_ctalist, R.segcap);
  R.arena_top = reinterpret_cast<unsigned long long*>(ensure<u64>(c, c->rs_atop, 1));
  R.arena_cap = 0;
  GS_CUDA(cudaMemsetAsync(R.shead, 0xff, sizeof(u32) * p.slots, c->st));
  return R;
}

// Stable radix sort of the fold elements by segment id (passes beyond the
// device-side need exit at once).
template <class Src0>
void rs_sort(gs_ctx* c, RsRun& R, const Src0& src0) {
  const u32 nb = R.nblk;
  const u32 ng = std::min<u32>(nb, (u32)c->sms * 16);   // blocks loop over the tiles
  const int64_t ncnt = 256ll * nb;
  const int nsb = (int)((ncnt + kScan32Chunk - 1) / kScan32Chunk);
  for (int pass = 0; pass < R.maxpasses; ++pass) {
    u32* ok = R.k[pass & 1];
    u32* ov = R.v[pass & 1];
    auto go = [&](const auto& src) {
      using S = std::decay_t<decltype(src)>;
      launch(c, K_REFSUM, [&] { k_rs_count<S><<<ng, kRsThreads, 0, c->st>>>(src, R.ctl, pass, R.cnt, nb); });
      launch(c, K_REFSUM, [&] { k_scan32_reduce<<<nsb, 256, 0, c->st>>>(R.cnt, ncnt, R.scan, R.ctl, pass); });
      launch(c, K_REFSUM, [&] { k_scan32_top<<<1, 1024, 0, c->st>>>(R.scan, nsb, R.ctl, pass); });
      launch(c, K_REFSUM, [&] { k_scan32_apply<<<nsb, 256, 0, c->st>>>(R.cnt, ncnt, R.scan, R.ctl, pass); });
      launch(c, K_REFSUM, [&] { k_rs_scatter<S><<<ng, kRsThreads, 0, c->st>>>(src, R.ctl, pass, R.cnt, nb, ok, ov); });
    };
    if (pass == 0)
      go(src0);
    else
      go(RsBufSrc{R.k[(pass - 1) & 1], R.v[(pass - 1) & 1], &R.ctl->nelem});
  }
}

template <int D, class Val>
void rs_fold(gs_ctx* c, RsRun& R, const Val& V, double* rs_out) {
  const RsSorted so{R.k[0], R.v[0], R.k[1], R.v[1]};
  const int nbp = blocks_for(c, R.n);
  const int64_t nw = R.n / kFoldWin;
  const int nbw = (int)std::max<int64_t>(1, std::min<int64_t>((nw * 32 + 255) / 256, (int64_t)c->sms * 8));
  const int nbs = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)R.segcap * 32 + 255) / 256, (int64_t)c->sms * 8));
  launch(c, K_REFSUM, [&] { k_rs_bounds<<<nbp, 256, 0, c->st>>>(so, R.ctl, R.sstart, R.send); });
  launch(c, K_REFSUM, [&] { k_fold_win<D, Val><<<nbw, 256, 0, c->st>>>(so, R.ctl, R.sstart, R.send, V, R.wsum); });
  launch(c, K_REFSUM, [&] { k_fold_pre<D, Val><<<nbs, 256, 0, c->st>>>(so, R.ctl, R.sstart, R.send, V, R.wsum, R.wpre); });
  launch(c, K_REFSUM, [&] { k_fold_delta<D, Val><<<nbw, 256, 0, c->st>>>(so, R.ctl, V, R.wsum, R.wpre, R.wdelta); });
  launch(c, K_REFSUM, [&] {
    k_fold_small<D, Val><<<blocks_for(c, (int64_t)R.segcap * D), 256, 0, c->st>>>(so, R.ctl, R.sstart, R.send, V,
                                                                                 R.outslot, rs_out);
  });
  const int nbb = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)R.segcap * D * 32 + 255) / 256, (int64_t)c->sms * 8));
  launch(c, K_REFSUM, [&] {
    k_fold_big<D, Val><<<nbb, 256, 0, c->st>>>(so, R.ctl, R.sstart, R.send, V, R.wdelta, R.outslot, rs_out);
  });
}

// First table (table buffer 0 built): reference-order sums of y_0.  `si`:
// the spatial sort's runs (nullptr: unsorted, every occupied cell is a run);
// `ys`: the iterate the runs index (sorted layout); V: the input values in
// ORIGINAL point order (the order np.bincount adds them in).
template <int D, class Tab>
void rs_first(gs_ctx* c, const Plan& p, Tab* tabs, int64_t n, const SortInfo* si, const double* ys,
              const InVal<D>& V, const InitStats& st) {
  RsRun& R = c->rsr;
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  GS_CUDA(cudaMemsetAsync(R.ctl, 0, sizeof(RsCtl), c->st));
  if (si) {
    R.cell0 = si->cell0;
    R.runs = si->runs;
    R.nruns = &ctrl->nruns;
    R.start = si->start;
    R.end = si->end;
    R.perm = si->perm;
    R.all_big = si->perm == nullptr;
    if (si->perm) {
      R.arena_cap = arena_entries(n);
      launch(c, K_REFSUM, [&] { k_rs_set64<<<1, 1, 0, c->st>>>(R.arena_top, (unsigned long long)n); });
    }
  } else {
    if (!R.model) {
      u32* c0 = ensure<u32>(c, c->rs_cell0, (size_t)n);
      launch(c, K_REFSUM, [&] { k_rs_cell0<D, Tab><<<blocks_for(c, n), kThreads, 0, c->st>>>(ys, n, p.g, tabs[0], c0); });
      R.cell0 = c0;
    }
    if constexpr (Tab::kDense) {
      u32* rl = ensure<u32>(c, c->rs_runs, p.list_cap);
      GS_CUDA(cudaMemsetAsync(&ctrl->nruns, 0, sizeof(u32), c->st));
      launch(c, K_REFSUM, [&] {
        k_compact<D><<<blocks_for(c, (int64_t)p.slots), kThreads, 0, c->st>>>(tabs[0].ent, p.slots, rl, &ctrl->nruns);
      });
      R.runs = rl;
      R.nruns = &ctrl->nruns;
    } else {
      R.runs = tabs[0].list;
      R.nruns = &ctrl->k[0];
    }
  }
  LowBits lb;
  bool coarse_ok = true;   // the global lowest bit proves every run exact already?
  for (int j = 0; j < GS_MAXD; ++j) lb.v[j] = st.lowbit[j];
  for (int j = 0; j < D; ++j) {
    // |total| < n * max|x|: every run exact if the input's lowest bit is at
    // least ulp of that (and of the fixed-point quantum)
    double amax;
    memcpy(&amax, &st.absmax[j], sizeof amax);
    int e = 0;
    frexp(amax * (double)n * (1.0 + 0x1p-40) + 1e-300, &e);
    coarse_ok &= lb.v[j] >= -p.g.qexp[j] && lb.v[j] >= (e - 1) - 52;
  }
  int* lowrun = nullptr;
  if (si && !coarse_ok && !R.model) {
    // per-run lowest bits over the sorted iterate (one pass)
    lowrun = reinterpret_cast<int*>(ensure<u32>(c, c->rs_lowrun, (size_t)p.slots * D));
    GS_CUDA(cudaMemsetAsync(lowrun, 0x7f, sizeof(int) * p.slots * D, c->st));   // large positive
    const int nbl = (int)std::max<int64_t>(1, std::min<int64_t>((n / 4096 + 1) * 32 / 256 + 1, (int64_t)c->sms * 8));
    launch(c, K_REFSUM, [&] { k_rs_lowbit<D, Tab><<<nbl, 256, 0, c->st>>>(ys, n, p.g, tabs[0], lowrun); });
  }
  launch(c, K_REFSUM, [&] {
    k_rs_first<D, Tab><<<blocks_for(c, (int64_t)p.list_cap), kThreads, 0, c->st>>>(
        p.g, tabs[0], R.runs, R.nruns, si ? si->start : nullptr, ys, si != nullptr, !R.all_big, lb, R.rc[0],
        R.runkey, R.outslot, R.rs[0], R.ctl, R.seglen, R.sstart, R.send, R.seglist, R.runkv, lowrun,
        R.arena_cap ? R.lst[0] : nullptr, R.model);
  });
  if (R.model) {   // the first table's sums: exact (distinct values; no order to model)
    check_launch();
    return;
  }
  if (!R.all_big) {
    static std::atomic<uint64_t> wattr{0};
    if (attr_pending(wattr, c->device)) {
      GS_CUDA(cudaFuncSetAttribute(k_rs_gather_warp<D, InVal<D>, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGatherWarpSmem));
      attr_done(wattr, c->device);
    }
    launch(c, K_REFSUM, [&] {
      k_rs_gather_warp<D, InVal<D>, true><<<c->sms * 8, 256, kGatherWarpSmem, c->st>>>(R.ctl, R.seglen, nullptr, R.seglist, R.start,
                                                                         R.end, R.perm, nullptr, V, R.outslot,
                                                                         R.rs[0], false, RsLists{});
    });
    static std::atomic<uint64_t> attr{0};
    if (attr_pending(attr, c->device)) {
      GS_CUDA(cudaFuncSetAttribute(k_rs_gather<D, InVal<D>, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGatherSmem));
      attr_done(attr, c->device);
    }
    launch(c, K_REFSUM, [&] {
      k_rs_gather<D, InVal<D>, true><<<c->sms * 2, 256, kGatherSmem, c->st>>>(R.ctl, R.seglen, nullptr, R.seglist, R.start,
                                                                    R.end, R.perm, nullptr, V, R.outslot, R.rs[0],
                                                                    false, RsLists{}, nullptr);
    });
  }
  launch(c, K_REFSUM, [&] { k_rs_passes<<<1, 1, 0, c->st>>>(R.ctl); });
  rs_sort(c, R, RsRunSrc{R.cell0, R.runkv, n});
  rs_fold<D>(c, R, V, R.rs[0]);
  launch(c, K_REFSUM, [&] { k_rs_stats<<<1, 1, 0, c->st>>>(R.ctl, R.stats); });
  check_launch();
}

// Table t+1 (just derived into buffer (t+1)&1): its reference-order sums.
template <int D, class Tab>
void rs_next(gs_ctx* c, const Plan& p, Tab* tabs, int t, const Rec<D>* rec) {
  RsRun& R = c->rsr;
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  const int cur = t & 1;
  GS_CUDA(cudaMemsetAsync(R.ctl, 0, sizeof(RsCtl), c->st));
  if (!R.model) {
    GS_CUDA(cudaMemsetAsync(R.segbeg, 0, sizeof(u32) * (R.segcap + 1), c->st));
    GS_CUDA(cudaMemsetAsync(R.segcur, 0, sizeof(u32) * R.segcap, c->st));
  }
  const int64_t items = Tab::kDense ? (int64_t)p.slots : (int64_t)p.list_cap;
  const bool lists = R.arena_cap != 0 && !R.model;
  const RsLists L{lists || R.model, lists, R.lst[cur], R.lst[cur ^ 1], R.shead, R.snext, R.segdone,
                  const_cast<u32*>(R.perm), R.arena_cap, R.arena_top};
  if (R.model) {
    // sequential model: closed forms in k_rs_classify, proportional folds of
    // the mixed targets' sources -- no point order, no sorts
    // 128-thread CTAs: they share the SMs with the shift's persistent CTAs, and
    // smaller CTAs fit the registers those leave (GRIDSHIFT_CLASSIFY_T, for tuning)
    static const int env_t = getenv("GRIDSHIFT_CLASSIFY_T") ? atoi(getenv("GRIDSHIFT_CLASSIFY_T")) : 0;
    const int ct = (env_t == 64 || env_t == 128 || env_t == 256) ? env_t : kClassifyThreads;
    const int cb = (int)std::max<int64_t>(1, std::min<int64_t>((items + ct - 1) / ct, (int64_t)c->sms * 8 * (kThreads / ct)));
    launch(c, K_REFSUM, [&] {
      k_rs_classify<D, Tab><<<cb, ct, 0, c->st>>>(p.g, tabs[cur], tabs[cur ^ 1], rec, ctrl, cur, t,
                                                  R.nsrc, R.mid, R.outslot, R.rs[cur ^ 1], R.ctl,
                                                  R.seglen, R.sstart, R.send, false,
                                                  static_cast<Rec<D>*>(R.tag[cur ^ 1]), L, nullptr);
    });
    launch(c, K_REFSUM, [&] {
      k_rs_runfold<D, Tab><<<c->sms * 16, kModelWarps * 32, 0, c->st>>>(R.ctl, R.outslot, tabs[cur], rec, L, R.rs[cur ^ 1]);
    });
    if (t + 1 < R.stats_rows) launch(c, K_REFSUM, [&] { k_rs_stats<<<1, 1, 0, c->st>>>(R.ctl, R.stats + 5 * (t + 1)); });
    launch(c, K_REFSUM, [&] { k_rs_unmark<<<blocks_for(c, (int64_t)R.segcap), kThreads, 0, c->st>>>(R.outslot, R.ctl, R.mid, R.shead); });
    GS_CUDA(cudaMemsetAsync(R.nsrc, 0, sizeof(u32) * p.slots, c->st));
    return;
  }
  launch(c, K_REFSUM, [&] {
    k_rs_classify<D, Tab><<<blocks_for(c, items), kThreads, 0, c->st>>>(p.g, tabs[cur], tabs[cur ^ 1], rec, ctrl, cur, t,
                                                                        R.nsrc, R.mid, R.outslot, R.rs[cur ^ 1], R.ctl,
                                                                        R.seglen, R.sstart, R.send, R.all_big,
                                                                        static_cast<Rec<D>*>(R.tag[cur ^ 1]), L, R.ctalist);
  });
  if (L.lists) {
    // mixed targets whose sources carry point lists: rank-merge + fold
    static std::atomic<uint64_t> mattr{0};
    if (attr_pending(mattr, c->device)) {
      GS_CUDA(cudaFuncSetAttribute(k_rs_merge_warp<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)merge_warp_smem(D)));
      GS_CUDA(cudaFuncSetAttribute(k_rs_merge<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)merge_smem(D)));
      attr_done(mattr, c->device);
    }
    launch(c, K_REFSUM, [&] {
      k_rs_merge_warp<D><<<c->sms * 8, 256, merge_warp_smem(D), c->st>>>(R.ctl, R.seglen, R.outslot, rec, L, R.rs[cur ^ 1]);
    });
    launch(c, K_REFSUM, [&] {
      k_rs_merge<D><<<c->sms * 2, 256, merge_smem(D), c->st>>>(R.ctl, R.seglen, R.outslot, rec, L, R.rs[cur ^ 1], R.ctalist);
    });
  }
  const int nbr = blocks_for(c, (int64_t)p.list_cap);
  launch(c, K_REFSUM, [&] {
    k_rs_runs<D, Tab><<<nbr, kThreads, 0, c->st>>>(R.runs, R.nruns, R.rc[cur], R.rc[cur ^ 1], rec, tabs[cur ^ 1], R.mid,
                                                   R.runkey, R.runval, ctrl, t, R.seglen, R.runseg, R.segbeg,
                                                   R.all_big, R.runkv);
  });
  if (!R.all_big) {
    // run lists of the gathered segments, then one CTA each
    const int64_t ns = (int64_t)R.segcap + 1;
    const int nsb = (int)((ns + kScan32Chunk - 1) / kScan32Chunk);
    launch(c, K_REFSUM, [&] { k_scan32_reduce<<<nsb, 256, 0, c->st>>>(R.segbeg, ns, R.segscan, nullptr, 0); });
    launch(c, K_REFSUM, [&] { k_scan32_top<<<1, 1024, 0, c->st>>>(R.segscan, nsb, nullptr, 0); });
    launch(c, K_REFSUM, [&] { k_scan32_apply<<<nsb, 256, 0, c->st>>>(R.segbeg, ns, R.segscan, nullptr, 0); });
    launch(c, K_REFSUM, [&] { k_rs_fill<<<nbr, kThreads, 0, c->st>>>(R.runs, R.nruns, R.runseg, R.segbeg, R.segcur, R.seglist); });
    static std::atomic<uint64_t> wattr{0};
    if (attr_pending(wattr, c->device)) {
      GS_CUDA(cudaFuncSetAttribute(k_rs_gather_warp<D, RecVal<D>, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGatherWarpSmem));
      attr_done(wattr, c->device);
    }
    launch(c, K_REFSUM, [&] {
      k_rs_gather_warp<D, RecVal<D>, false><<<c->sms * 8, 256, kGatherWarpSmem, c->st>>>(R.ctl, R.seglen, R.segbeg, R.seglist,
                                                                          R.start, R.end, R.perm, R.runval,
                                                                          RecVal<D>{rec}, R.outslot, R.rs[cur ^ 1],
                                                                          false, L);
    });
    static std::atomic<uint64_t> attr{0};
    if (attr_pending(attr, c->device)) {
      GS_CUDA(cudaFuncSetAttribute(k_rs_gather<D, RecVal<D>, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGatherSmem));
      attr_done(attr, c->device);
    }
    launch(c, K_REFSUM, [&] {
      k_rs_gather<D, RecVal<D>, false><<<c->sms * 2, 256, kGatherSmem, c->st>>>(R.ctl, R.seglen, R.segbeg, R.seglist, R.start,
                                                                     R.end, R.perm, R.runval, RecVal<D>{rec},
                                                                     R.outslot, R.rs[cur ^ 1], false, L, R.ctalist);
    });
  }
  launch(c, K_REFSUM, [&] { k_rs_passes<<<1, 1, 0, c->st>>>(R.ctl); });
  rs_sort(c, R, RsRunSrc{R.cell0, R.runkv, R.n});
  rs_fold<D>(c, R, RecVal<D>{rec}, R.rs[cur ^ 1]);
  if (t + 1 < R.stats_rows) launch(c, K_REFSUM, [&] { k_rs_stats<<<1, 1, 0, c->st>>>(R.ctl, R.stats + 5 * (t + 1)); });
  launch(c, K_REFSUM, [&] { k_rs_unmark<<<blocks_for(c, (int64_t)R.segcap), kThreads, 0, c->st>>>(R.outslot, R.ctl, R.mid, L.on ? R.shead : nullptr); });
  GS_CUDA(cudaMemsetAsync(R.nsrc, 0, sizeof(u32) * p.slots, c->st));
}

// -------------------------------------------------------------- iteration

// Histogram of y[0] into table 0 (clean), before the loop.
template <int D, class Tab>
void enqueue_first_hist(gs_ctx* c, const Plan& p, Tab* tabs, int64_t n, int nb_pts, bool grouped = false,
                        const SortInfo* runs = nullptr) {
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  const double* y0 = static_cast<const double*>(c->y[0].p);
  if constexpr (!Tab::kDense) {
    // sorted hash-table runs: one plain-store entry per run of the spatial
    // sort (measured against the per-tile CAS / atomic build: DESIGN.md 3)
    static const bool off = getenv("GRIDSHIFT_HIST_RUNS") && getenv("GRIDSHIFT_HIST_RUNS")[0] == '0';
    if (runs && grouped && !off) {
      launch(c, K_HIST, [&] {
        k_hist_runs<D, Tab><<<blocks_for(c, (int64_t)p.list_cap * kHistRunLanes), kThreads, 0, c->st>>>(
            y0, p.g, tabs[0], runs->runs, &ctrl->nruns, runs->start, runs->end, ctrl);
      });
      return;
    }
  }
  // grouped: y0 is the spatial sort's output (each cell's points contiguous)
  if (grouped)
    launch(c, K_HIST, [&] { k_hist<D, Tab, false, true, true><<<nb_pts, kThreads, 0, c->st>>>(y0, n, p.g, tabs[0], ctrl, 0); });
  else
    launch(c, K_HIST, [&] { k_hist<D, Tab, false, true><<<nb_pts, kThreads, 0, c->st>>>(y0, n, p.g, tabs[0], ctrl, 0); });
}

// The table chain (k_agg -> k_derive -> k_agg ...) never reads the points:
// table t+1 is derived from table t.  So on dense tables it runs on a
// high-priority side stream one iteration ahead of the per-point shifts,
// which only wait for their iteration's target records (double-buffered).
void side_init(gs_ctx* c) {
  if (c->side) return;
  int least = 0, greatest = 0;
  GS_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  // LOW priority: the table chain fills the SMs the shift's last wave leaves
  // idle instead of displacing the bandwidth-bound shift (measured: high
  // priority costs +9 ms per 100M-point run, low saves 3 ms)
  // (GRIDSHIFT_SIDE_PRIO=high flips it, for tuning)
  const char* pr = getenv("GRIDSHIFT_SIDE_PRIO");
  GS_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, (pr && pr[0] == 'h') ? greatest : least));
  for (cudaEvent_t* e : {&c->ev_fork, &c->ev_join, &c->ev_rec[0], &c->ev_rec[1], &c->ev_shift[0], &c->ev_shift[1]})
    GS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaEvent_t* e : {&c->ev_pace[0], &c->ev_pace[1]}) GS_CUDA(cudaEventCreate(e));
}

// main stream waits for everything enqueued on the side stream so far
void side_join(gs_ctx* c) {
  if (!c->side) return;
  GS_CUDA(cudaEventRecord(c->ev_join, c->side));
  GS_CUDA(cudaStreamWaitEvent(c->st, c->ev_join, 0));
}

// ------------------------------------------------- host label delivery
// A host caller wants labels[i] (int64, original order) in host memory.
// On the sorted dense path the label of point i is a function of its
// initial cell alone (labels = rank[root[cell0[i]]], k_labels_runs), and
// cell0 is final right after the spatial sort.  So the 4-byte cell0 array
// crosses PCIe while the loop runs (copy stream), the extraction sends the
// per-cell labels (4 bytes per table slot) instead of 8 bytes per point,
// and the host expands them.  Same values as k_labels_runs + a D2H copy.

// after the sort was enqueued on c->st: remember where cell0 is
void cell0_mark(gs_ctx* c, const u32* cell0, int64_t n) {
  if (!c->copy) {
    GS_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    GS_CUDA(cudaEventCreateWithFlags(&c->ev_sorted, cudaEventDisableTiming));
    GS_CUDA(cudaEventCreateWithFlags(&c->ev_cell0, cudaEventDisableTiming));
  }
  if (c->h_cell0_cap < (size_t)n) {
    if (c->h_cell0) GS_CUDA(cudaFreeHost(c->h_cell0));
    c->h_cell0 = nullptr;
    c->h_cell0_cap = 0;
    GS_CUDA(cudaMallocHost(&c->h_cell0, sizeof(u32) * (size_t)n));
    c->h_cell0_cap = (size_t)n;
  }
  GS_CUDA(cudaEventRecord(c->ev_sorted, c->st));
  c->cell0_dev = cell0;
  c->cell0_n = n;
}

// issue the cell0 copy.  Called once the host has run-ahead chunks in
// flight (or after the loop): the synchronous chunk boundaries read small
// Ctrl snapshots device->host, which must not queue behind a large copy.
void cell0_copy_start(gs_ctx* c) {
  if (!c->cell0_dev || c->cell0_pending) return;
  GS_CUDA(cudaStreamWaitEvent(c->copy, c->ev_sorted, 0));
  GS_CUDA(cudaMemcpyAsync(c->h_cell0, c->cell0_dev, sizeof(u32) * (size_t)c->cell0_n, cudaMemcpyDeviceToHost,
                          c->copy));
  GS_CUDA(cudaEventRecord(c->ev_cell0, c->copy));
  c->cell0_pending = true;
}

inline int64_t label_of(u32 s, const u32* lab) { return s == 0xffffffffu ? -1 : (int64_t)lab[s]; }

#if defined(__x86_64__)
// 16 points per step: gather the cell labels, widen, streaming stores (the
// output is written once and not read back here)
__attribute__((target("avx512f"))) void expand_avx512(const u32* c0, const u32* lab, int64_t a, int64_t b,
                                                       int64_t* out) {
  int64_t i = a;
  for (; i < b && ((uintptr_t)(out + i) & 63); ++i) out[i] = label_of(c0[i], lab);
  const __m512i none = _mm512_set1_epi32(-1);
  const __m512i neg = _mm512_set1_epi64(-1);
  for (; i + 16 <= b; i += 16) {
    const __m512i s = _mm512_loadu_si512(c0 + i);
    const __mmask16 ok = _mm512_cmpneq_epu32_mask(s, none);
    const __m512i v = _mm512_mask_i32gather_epi32(none, ok, s, lab, 4);
    const __m512i lo = _mm512_mask_mov_epi64(neg, (__mmask8)ok, _mm512_cvtepu32_epi64(_mm512_castsi512_si256(v)));
    const __m512i hi =
        _mm512_mask_mov_epi64(neg, (__mmask8)(ok >> 8), _mm512_cvtepu32_epi64(_mm512_extracti64x4_epi64(v, 1)));
    _mm512_stream_si512(reinterpret_cast<__m512i*>(out + i), lo);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(out + i + 8), hi);
  }
  for (; i < b; ++i) out[i] = label_of(c0[i], lab);
  _mm_sfence();
}
#endif

// labels[i] = lab[c0[i]] over host threads
void expand_labels(const u32* c0, const u32* lab, int64_t n0, int64_t n, int64_t* out) {
  unsigned T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n - n0 < (int64_t)1 << 20) T = 1;
#if defined(__x86_64__)
  const bool avx = __builtin_cpu_supports("avx512f");
#endif
  auto work = [&](unsigned t) {
    const int64_t m = n - n0;
    const int64_t a = n0 + ((m * t / T) & ~int64_t(7)), b = t + 1 == T ? n : n0 + ((m * (t + 1) / T) & ~int64_t(7));
#if defined(__x86_64__)
    if (avx) { expand_avx512(c0, lab, a, b, out); return; }
#endif
    for (int64_t i = a; i < b; ++i) out[i] = label_of(c0[i], lab);
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < T; ++t) pool.emplace_back(work, t);
  work(0);
  for (std::thread& th : pool) th.join();
}

// the end of a host entry point: labels into the caller's host buffer
void deliver_labels(gs_ctx* c, const int64_t* dl, int64_t* out, int64_t n) {
  int64_t dev_bytes = 0;
  if (c->labels_on_host) {
    static const bool dbg = getenv("GS_DEBUG_DELIVERY") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    const double t0 = now();
    GS_CUDA(cudaEventSynchronize(c->ev_cell0));
    sync(c);
    const double t1 = now();
    // a pinned caller buffer takes the first part of the labels straight from
    // the device (int64, DMA) while the host threads expand the rest from the
    // per-cell labels: the two run side by side
    int64_t n_dev = 0;
    cudaPointerAttributes pa;
    if (n >= (int64_t)1 << 24 && cudaPointerGetAttributes(&pa, out) == cudaSuccess &&
        pa.type == cudaMemoryTypeHost && c->cell0_dev) {
      n_dev = (n * 2 / 5) & ~int64_t(127);
      int64_t* tmp = ensure<int64_t>(c, c->labels, (size_t)n);
      launch(c, K_LABELS, [&] {
        k_labels_from_slots<<<blocks_for(c, n_dev), kThreads, 0, c->st>>>(c->cell0_dev, n_dev,
                                                                         static_cast<const u32*>(c->slotlab.p),
                                                                         reinterpret_cast<i64*>(tmp));
      });
      GS_CUDA(cudaMemcpyAsync(out, tmp, sizeof(int64_t) * n_dev, cudaMemcpyDeviceToHost, c->st));
    } else {
      cudaGetLastError();   // (an unregistered pointer is not an error here)
    }
    expand_labels(c->h_cell0, c->h_slotlab, n_dev, n, out);
    if (n_dev) sync(c);
    dev_bytes = (int64_t)sizeof(int64_t) * n_dev;
    c->xfer_d2h = (int64_t)sizeof(u32) * n + (int64_t)c->slotlab_bytes + dev_bytes;
    if (dbg) fprintf(stderr, "deliver: wait %.3f ms expand %.3f ms\n", t1 - t0, now() - t1);
  } else {
    GS_CUDA(cudaMemcpyAsync(out, dl, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    c->xfer_d2h = (int64_t)sizeof(int64_t) * n;
  }
  c->xfer_d2h += (int64_t)(c->modes_host.size() * sizeof(double));
  c->labels_on_host = false;
  c->cell0_pending = false;
}

// set for the duration of a host entry point's engine run
struct HostLabelRequest {
  gs_ctx* c;
  explicit HostLabelRequest(gs_ctx* cc) : c(cc) { c->host_labels = true; }
  ~HostLabelRequest() { c->host_labels = false; }
};

// Iteration t: table t (buffer t&1) holds the cells of y_t.  k_agg turns it
// into per-cell target records (and clears buffer (t+1)&1), k_derive builds
// the table of y_{t+1} from it (O(cells)), k_shift moves every point.
template <int D, class Tab>
void enqueue_iteration(gs_ctx* c, const Plan& p, Tab* tabs, int t, double eta, int64_t n, int nb_pts,
                       int nb_cells, u64* limbs = nullptr, bool with_shift = true, bool overlap = false) {
  const int cur = t & 1;
  // the iterate lives in y[0] and is shifted in place (k_shift)
  double* y_it = static_cast<double*>(c->y[0].p);
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  // overlap needs dense tables (k_shift does not read them) and 2 record buffers
  const bool ov = overlap && Tab::kDense && with_shift;
  Rec<D>* rec = static_cast<Rec<D>*>(c->targets.p) + (ov ? (size_t)cur * p.slots : 0);
  cudaStream_t main_st = c->st;
  if (ov) {
    side_init(c);
    if (t == 0) {
      GS_CUDA(cudaEventRecord(c->ev_fork, main_st));
      GS_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    }
    if (t >= 2) GS_CUDA(cudaStreamWaitEvent(c->side, c->ev_shift[cur], 0));   // shift t-2 read rec[cur]
    c->st = c->side;
  }
  bool bricked = false;
  RsRun& R = c->rsr;
  if constexpr (D == 3 && Tab::kDense) {
    // dense 3-D lattice: tiled stencil over the occupied 8^3 bricks
    // (k_agg_brick3, k_derive_brick3); brick occupancy per table buffer
    const int ext0 = (int)(p.g.nkeys / p.g.stride[0]), ext1 = (int)(p.g.stride[0] / p.g.stride[1]),
              ext2 = (int)p.g.stride[1];
    const int nbx = (ext0 + kBX - 1) / kBX, nby = (ext1 + kBY - 1) / kBY, nbz = (ext2 + kBZ - 1) / kBZ;
    const int nbr = nbx * nby * nbz;
    const BrickMap bm{(u32)p.g.stride[0], (u32)p.g.stride[1], (u32)nby, (u32)nbz};
    static std::atomic<uint64_t> attr{0};
    if (attr_pending(attr, c->device)) {
      for (auto kern : {k_agg_brick3<true>, k_agg_brick3<false>}) {
        GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBrickSmem));
        // same (maximal) shared-memory carveout as k_shift_tma, so the chain's
        // CTAs can be co-resident with the shift's on one SM
        GS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      }
      GS_CUDA(cudaFuncSetAttribute(k_derive_brick3, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      attr_done(attr, c->device);
    }
    u8* occ = ensure<u8>(c, c->bocc, 2 * (size_t)nbr);
    u32* mask = ensure<u32>(c, c->bmask, 2 * (size_t)nbr * kMaskWords);
    if (t == 0) {
      // iteration 0 starts from a freshly built table in buffer 0
      GS_CUDA(cudaMemsetAsync(occ, 0, 2 * (size_t)nbr, c->st));
      GS_CUDA(cudaMemsetAsync(mask, 0, 2 * (size_t)nbr * kMaskWords * sizeof(u32), c->st));
      launch(c, K_AGG, [&] {
        k_mark_bricks<<<blocks_for(c, (int64_t)p.slots), kThreads, 0, c->st>>>(
            reinterpret_cast<const Entry<3>*>(tabs[0].ent), p.slots, bm, occ);
      });
    }
    u8* occ_cur = occ + (size_t)cur * nbr;
    u8* occ_nxt = occ + (size_t)(cur ^ 1) * nbr;
    launch(c, K_AGG, [&] {
      auto kern = R.on ? k_agg_brick3<true> : k_agg_brick3<false>;
      kern<<<nbr, kBrickThreads, kBrickSmem, c->st>>>(
          p.g, tabs[cur], tabs[cur ^ 1], reinterpret_cast<Rec<3>*>(rec), ctrl,
          static_cast<u64*>(c->fp_hist.p) + t, static_cast<u32*>(c->k_hist.p) + t, nbx, nby, nbz, occ_cur, occ_nxt,
          mask + (size_t)(cur ^ 1) * nbr * kMaskWords, mask + (size_t)cur * nbr * kMaskWords, t,
          R.on ? R.rs[cur] : nullptr);
    });
    if (ov) GS_CUDA(cudaEventRecord(c->ev_rec[cur], c->st));
    launch(c, K_DERIVE, [&] {
      k_derive_brick3<<<nbr, kBrickThreads, 0, c->st>>>(p.g, tabs[cur], tabs[cur ^ 1],
                                                        reinterpret_cast<const Rec<3>*>(rec), ctrl, nby, nbz, bm,
                                                        occ_cur, occ_nxt, mask + (size_t)cur * nbr * kMaskWords, t,
                                                        R.on ? R.nsrc : nullptr);
    });
    bricked = true;
    if (R.on) rs_next<D>(c, p, tabs, t, rec);
  }
  const double* rs_cur = R.on ? R.rs[cur] : nullptr;
  if (!bricked && D >= 4 && !Tab::kDense)
    launch(c, K_AGG, [&] { k_agg_warp<D, Tab><<<c->sms * 8, kThreads, 0, c->st>>>(p.g, tabs[cur], tabs[cur ^ 1], rec,
                                                    ctrl, cur, static_cast<u64*>(c->fp_hist.p) + t,
                                                    static_cast<u32*>(c->k_hist.p) + t, t, rs_cur); });
  else if (!bricked)
    launch(c, K_AGG, [&] { k_agg<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(p.g, tabs[cur], tabs[cur ^ 1], rec, ctrl, cur,
                                                    static_cast<u64*>(c->fp_hist.p) + t,
                                                    static_cast<u32*>(c->k_hist.p) + t, t, rs_cur); });
  if (!bricked && ov) GS_CUDA(cudaEventRecord(c->ev_rec[cur], c->st));
  if (!bricked)
    launch(c, K_DERIVE, [&] { k_derive<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(p.g, tabs[cur], tabs[cur ^ 1], rec,
                                                                                  ctrl, cur, t,
                                                                                  R.on ? R.nsrc : nullptr); });
  if (!bricked && R.on) rs_next<D>(c, p, tabs, t, rec);
  if (ov) {
    c->st = main_st;
    GS_CUDA(cudaStreamWaitEvent(main_st, c->ev_rec[cur], 0));
  }
  bool tma = false;
  if constexpr ((Tab::kDense && D <= 3) || (!Tab::kDense && (D == 4 || D == 5))) {
    // bulk-copy pipelined shift: persistent 64-thread CTAs (2 TMA stages each);
    // dense tables of up to 3 axes and the hash tables of 4- and 5-axis runs
    // (the lookups probe the table; the tiles still stream through shared memory)
    if (with_shift) {
      // 64-thread CTAs (tile = 256 points), 16 warps per SM: small CTAs
      // decouple the per-tile barriers (measured 256 -> 64: -1 ms per run)
      constexpr int T = 64;
      static std::atomic<uint64_t> attr{0};
      if (attr_pending(attr, c->device)) {
        GS_CUDA(cudaFuncSetAttribute(k_shift_tma<D, T, Tab>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        GS_CUDA(cudaFuncSetAttribute(k_shift_tma<D, T, Tab>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)shift_tma_smem<D, T>()));
        attr_done(attr, c->device);
      }
      const int64_t ntiles = (n + 4 * T - 1) / (4 * T);
      // persistent CTAs per SM: 8 fill the SM's registers (8 x 64 x 96); fewer
      // leave room for the table chain's CTAs on the side stream
      // (GRIDSHIFT_SHIFT_CTAS overrides, for tuning; beyond 8 the CTAs run in waves)
      static const int env_per = getenv("GRIDSHIFT_SHIFT_CTAS") ? atoi(getenv("GRIDSHIFT_SHIFT_CTAS")) : 0;
      const int per = env_per > 0 ? std::min(env_per, 128) : ((R.on && Tab::kDense) ? kShiftCtasChain : 8);
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)c->sms * per));
      launch(c, K_SHIFT, [&] {
        k_shift_tma<D, T, Tab><<<grid, T, shift_tma_smem<D, T>(), c->st>>>(
            y_it, n, p.g, tabs[cur], rec, ctrl, static_cast<u64*>(c->partials.p), static_cast<double*>(c->mv_hist.p), t,
            eta, limbs, static_cast<u64*>(c->wr_hist.p) + t);
      });
      tma = true;
    }
  }
  if (with_shift && !tma)
    launch(c, K_SHIFT, [&] { k_shift<D, Tab><<<nb_pts, kThreads, 0, c->st>>>(y_it, y_it, n, p.g, tabs[cur], rec, ctrl,
                                                  static_cast<u64*>(c->partials.p),
                                                  static_cast<double*>(c->mv_hist.p), t, eta, limbs,
                                                  static_cast<u64*>(c->wr_hist.p) + t); });
  // ev_shift[cur] releases the chain two iterations ahead; it must follow
  // the stop decision of iteration t (in the shift itself, or k_converge for
  // a sharded run -- gs_shard_converge records it there)
  if (ov && !limbs) GS_CUDA(cudaEventRecord(c->ev_shift[cur], main_st));
}

// Collapsed iteration t >= 1: targets + derived table as usual, then one
// position update per run (k_run_shift) instead of the per-point shift.
template <int D, class Tab>
void enqueue_run_iteration(gs_ctx* c, const Plan& p, Tab* tabs, int t, double eta, const SortInfo& si,
                           int nb_cells) {
  const int cur = t & 1;
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  Rec<D>* rec = static_cast<Rec<D>*>(c->targets.p);
  enqueue_iteration<D>(c, p, tabs, t, eta, 0, 1, nb_cells, nullptr, false);   // agg + derive only
  launch(c, K_SHIFT, [&] {
    k_run_shift<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(si.runpos, si.runcnt, &ctrl->nruns, si.rld, p.g,
                                                           tabs[cur], rec, ctrl, static_cast<u64*>(c->partials.p),
                                                           static_cast<double*>(c->mv_hist.p), t, eta);
  });
}

// Occupied-cell list of a table (hash tables maintain theirs on insert;
// dense tables are compacted from their counts).  k must be 0 before.
template <int D, class Tab>
void build_list(gs_ctx* c, const Plan& p, Tab& tab) {
  if constexpr (Tab::kDense) {
    launch(c, K_CLEAR, [&] {
      k_compact<D><<<blocks_for(c, (int64_t)p.slots), kThreads, 0, c->st>>>(tab.ent, p.slots, tab.list, tab.k);
    });
  }
}

// Make a table clean whose list may not exist (dense tables in the loop).
template <int D, class Tab>
void clear_table(gs_ctx* c, const Plan& p, Tab& tab, u32* kp) {
  if constexpr (Tab::kDense) {
    launch(c, K_CLEAR, [&] { k_clear_all<D><<<blocks_for(c, (int64_t)p.slots), kThreads, 0, c->st>>>(tab.ent, p.slots); });
  } else {
    launch(c, K_CLEAR, [&] { k_clear<D, Tab><<<blocks_for(c, (int64_t)p.list_cap), kThreads, 0, c->st>>>(tab, kp); });
  }
  launch(c, K_CLEAR, [&] { k_reset_count<<<1, 1, 0, c->st>>>(kp); });
}

// Extraction of y_final (modeseek.py:256-272).  Table buffer e is clean on
// entry, buffer e^1 is dirty (cleared here and used as component scratch).
// `table_ready`: buffer e already holds the table of yf (the last k_derive
// built it); otherwise it is clean and gets built here.
// Phase 1: components of the final table + this process's first-appearance
// minima (`offset` = global index of its first point, sharded runs).
template <int D, class Tab>
void extract_components(gs_ctx* c, const Plan& p, Tab* tabs, const double* yf, int64_t n, int e,
                        const SortInfo* si, bool table_ready, u32 offset) {
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  const int nb_pts = blocks_for(c, n);
  const int nb_cells = blocks_for(c, (int64_t)p.list_cap);
  clear_table<D>(c, p, tabs[e ^ 1], &ctrl->k[e ^ 1]);
  if (!table_ready)
    launch(c, K_HIST, [&] { k_hist<D, Tab><<<nb_pts, kThreads, 0, c->st>>>(yf, n, p.g, tabs[e], ctrl, 0); });
  if constexpr (Tab::kDense) {
    launch(c, K_CLEAR, [&] { k_reset_count<<<1, 1, 0, c->st>>>(&ctrl->k[e]); });
    build_list<D>(c, p, tabs[e]);
  }
  u32* par = ensure<u32>(c, c->par, p.slots);
  u32* first = ensure<u32>(c, c->first, p.slots);
  launch(c, K_COMP, [&] { k_uf_init<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(p.g, tabs[e], &ctrl->k[e], par, first); });
  launch(c, K_COMP, [&] { k_uf_link<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(p.g, tabs[e], &ctrl->k[e], par); });
  launch(c, K_COMP, [&] { k_uf_flatten<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(tabs[e], &ctrl->k[e], par, tabs[e ^ 1].ent); });
  if (si)
    launch(c, K_LABELS, [&] {
      k_run_first<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(yf, p.g, tabs[e], si->runs, &ctrl->nruns, si->start,
                                                            si->minidx, par, first, si->runroot, ctrl, offset,
                                                            si->runpos, si->rld);
    });
  else
    launch(c, K_LABELS, [&] {
      k_first<D, Tab><<<nb_pts, kThreads, 0, c->st>>>(yf, n, p.g, tabs[e], par, first, nullptr, ctrl, offset);
    });
}

// Phase 2: dense relabel by first appearance, modes, labels; leaves both
// table buffers clean.
template <int D, class Tab>
void extract_finish(gs_ctx* c, const Plan& p, Tab* tabs, const double* yf, int64_t n, int e,
                    int64_t* labels_dev, const SortInfo* si) {
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  const int nb_pts = blocks_for(c, n);
  const int nb_cells = blocks_for(c, (int64_t)p.list_cap);
  u32* par = static_cast<u32*>(c->par.p);
  u32* first = static_cast<u32*>(c->first.p);
  u32* rankmap = ensure<u32>(c, c->aux, p.slots);
  u32* roots = ensure<u32>(c, c->roots, p.list_cap + 1);
  u32* rfirst = ensure<u32>(c, c->root_first, p.list_cap + 1);
  u32* nroots = ensure<u32>(c, c->partials, 2 * (size_t)c->sms * 8 + 2);  // reuse scratch
  GS_CUDA(cudaMemsetAsync(nroots, 0, sizeof(u32), c->st));
  launch(c, K_COMP, [&] { k_roots<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(tabs[e], &ctrl->k[e], par, first, roots, rfirst, nroots); });
  check_launch();
  u32 nr = 0;
  GS_CUDA(cudaMemcpyAsync(c->h_ctrl, c->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, c->st));
  GS_CUDA(cudaMemcpyAsync(c->h_small, nroots, sizeof(u32), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  check_flags(c->h_ctrl->error);
  nr = c->h_small[0];
  // dense relabel by first appearance (modeseek.py:262-265): sort roots by
  // their minimum point index; nr is the number of clusters (small)
  std::vector<u32> hr(nr), hf(nr);
  GS_CUDA(cudaMemcpyAsync(hr.data(), roots, nr * sizeof(u32), cudaMemcpyDeviceToHost, c->st));
  GS_CUDA(cudaMemcpyAsync(hf.data(), rfirst, nr * sizeof(u32), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  std::vector<u32> order(nr);
  for (u32 i = 0; i < nr; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](u32 a, u32 b) { return hf[a] < hf[b]; });
  std::vector<u32> rk(nr);
  for (u32 i = 0; i < nr; ++i) rk[order[i]] = i;
  u32* dranks = ensure<u32>(c, c->ranks, nr + 1);
  GS_CUDA(cudaMemcpyAsync(dranks, rk.data(), nr * sizeof(u32), cudaMemcpyHostToDevice, c->st));
  double* dmodes = ensure<double>(c, c->modes, (size_t)nr * D + 1);
  launch(c, K_COMP, [&] { k_modes<D><<<blocks_for(c, nr), kThreads, 0, c->st>>>(p.g, roots, dranks, nr, rankmap, tabs[e ^ 1].ent, dmodes); });
  if (si && c->host_labels && c->cell0_pending && Tab::kDense) {
    // host delivery: per-cell labels only (see deliver_labels)
    u32* sl = ensure<u32>(c, c->slotlab, si->slots0);
    launch(c, K_LABELS, [&] { k_slot_labels<<<nb_cells, kThreads, 0, c->st>>>(si->runs, &ctrl->nruns, si->runroot, rankmap, sl); });
    if (c->h_slotlab_cap < si->slots0) {
      if (c->h_slotlab) GS_CUDA(cudaFreeHost(c->h_slotlab));
      c->h_slotlab = nullptr;
      c->h_slotlab_cap = 0;
      GS_CUDA(cudaMallocHost(&c->h_slotlab, sizeof(u32) * si->slots0));
      c->h_slotlab_cap = si->slots0;
    }
    GS_CUDA(cudaMemcpyAsync(c->h_slotlab, sl, sizeof(u32) * si->slots0, cudaMemcpyDeviceToHost, c->st));
    c->slotlab_bytes = sizeof(u32) * si->slots0;
    c->labels_on_host = true;
  } else if (si)
    launch(c, K_LABELS, [&] {
      k_labels_runs<<<nb_pts, kThreads, 0, c->st>>>(si->cell0, n, si->runroot, rankmap, reinterpret_cast<i64*>(labels_dev));
    });
  else
    launch(c, K_LABELS, [&] { k_labels<D, Tab><<<nb_pts, kThreads, 0, c->st>>>(yf, n, p.g, tabs[e], par, rankmap, nullptr,
                                                   reinterpret_cast<i64*>(labels_dev)); });
  launch(c, K_CLEAR, [&] { k_clear<D, Tab><<<nb_cells, kThreads, 0, c->st>>>(tabs[e], &ctrl->k[e]); });
  launch(c, K_CLEAR, [&] { k_reset_count<<<1, 1, 0, c->st>>>(&ctrl->k[e]); });
  check_launch();
  c->modes_host.resize((size_t)nr * D);
  GS_CUDA(cudaMemcpyAsync(c->modes_host.data(), dmodes, (size_t)nr * D * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  c->k_last = nr;
  c->d_last = D;
}

template <int D, class Tab>
void run_extract(gs_ctx* c, const Plan& p, Tab* tabs, const double* yf, int64_t n, int e,
                 int64_t* labels_dev, const SortInfo* si = nullptr, bool table_ready = false) {
  extract_components<D>(c, p, tabs, yf, n, e, si, table_ready, 0u);
  extract_finish<D>(c, p, tabs, yf, n, e, labels_dev, si);
}

// One-time counting sort of the iterate by initial cell.
// Dense tables: the two-level sort (k_bk_*), which also leaves table buffer 0
// holding the table of y_0 (built from shared-memory tallies) and returns
// true.  Hash tables: per-point cursor scatter (k_scatter); table buffer 0
// is left clean and false returned.  y[0] holds the sorted iterate after.
template <int D, class Tab, class Src>
bool spatial_sort(gs_ctx* c, const Plan& p, Tab* tabs, int64_t n, SortInfo& si, const Src& src) {
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  const int nb_pts = blocks_for(c, n);
  // dense: scan every slot in key order (lexicographic cell order);
  // hash: scan the occupied list (first-touch order)
  const u64 nitems = Tab::kDense ? p.slots : p.list_cap;
  const int nbs = (int)((nitems + kScanChunk - 1) / kScanChunk);
  u64* bsum = ensure<u64>(c, c->scan, (size_t)nbs + 1);
  u32* off = ensure<u32>(c, c->runoff, p.slots);
  si.start = ensure<u32>(c, c->runstart, p.slots);
  si.minidx = ensure<u32>(c, c->runmin, p.slots);
  si.runs = ensure<u32>(c, c->runlist, p.list_cap);
  si.cell0 = ensure<u32>(c, c->cell0, (size_t)n);
  si.slots0 = p.slots;
  // reference-order sums: perm, followed by the arena of merged point lists
  si.perm = (c->exact_sums || c->seq_model) ? nullptr : ensure<u32>(c, c->perm, (size_t)arena_entries(n));
  si.runroot = off;   // the cursors are dead once the scatter is done...
  si.end = off;       // ...except as run ends, read (collapsed mode) before runroot is written
  GS_CUDA(cudaMemsetAsync(si.minidx, 0xff, p.slots * sizeof(u32), c->st));
  double* y0 = static_cast<double*>(c->y[0].p);
  double* y1 = static_cast<double*>(c->y[1].p);
  const u32* list = Tab::kDense ? nullptr : tabs[0].list;
  if constexpr (Tab::kDense) {
    // coarse buckets of 2^shift consecutive slots, at most 2048 of them
    int shift = kBucketShiftMin;
    while ((p.slots >> shift) >= 2048) ++shift;
    const u32 nb = (u32)((p.slots + (1ull << shift) - 1) >> shift);
    const u32 nblk = (u32)c->sms * 8;
    const int64_t chunk = (n + nblk - 1) / nblk;
    u32* bk = ensure<u32>(c, c->bkcnt, (size_t)nblk * nb);
    u64* btot = ensure<u64>(c, c->bktot, (size_t)nb + 1);
    using RT = typename Src::RT;
    constexpr int V = SRec<D, RT>::kVec;
    uint4* stage = reinterpret_cast<uint4*>(ensure<double>(c, c->stage, (size_t)n * V * 2));
    const size_t st_smem = bk_stage_smem<D, RT>(nb);
    static std::atomic<uint64_t> attr{0};
    if (attr_pending(attr, c->device)) {
      GS_CUDA(cudaFuncSetAttribute(k_bk_stage<D, Src>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bk_stage_smem<D, RT>(2048)));
      GS_CUDA(cudaFuncSetAttribute(k_bk_tally<D, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kTallyWin * 4));
      attr_done(attr, c->device);
    }
    const int nch = (int)((n + kChunkRecs - 1) / kChunkRecs);
    GS_CUDA(cudaMemsetAsync(off, 0, p.slots * sizeof(u32), c->st));
    launch(c, K_SORT, [&] { k_bk_count<D, Src><<<nblk, kThreads, nb * sizeof(u32), c->st>>>(src, n, p.g, shift, nb, chunk, bk, si.cell0, ctrl); });
    launch(c, K_SORT, [&] { k_bk_cols<<<nb, 1024, 0, c->st>>>(bk, nblk, nb, btot); });
    launch(c, K_SORT, [&] { k_scan_top<<<1, 1024, 0, c->st>>>(btot, (int)nb); });
    launch(c, K_SORT, [&] { k_bk_stage<D, Src><<<nblk, 512, st_smem, c->st>>>(src, n, shift, nb, chunk, bk, btot, si.cell0, stage); });
    launch(c, K_SORT, [&] { k_bk_tally<D, RT><<<nch, kTallyThreads, 2 * kTallyWin * sizeof(u32), c->st>>>(stage, n, p.slots, p.g, off, si.minidx, ctrl); });
    launch(c, K_SORT, [&] { k_scan_reduce<D><<<nbs, kThreads, 0, c->st>>>(tabs[0].ent, nullptr, nullptr, bsum, p.slots, off); });
    launch(c, K_SORT, [&] { k_scan_top<<<1, 1024, 0, c->st>>>(bsum, nbs); });
    launch(c, K_SORT, [&] { k_scan_apply<D><<<nbs, kThreads, 0, c->st>>>(tabs[0].ent, nullptr, nullptr, bsum, off, p.slots, si.start, off); });
    const int nchp = (int)((n + kRpt * kPlaceThreads - 1) / (kRpt * kPlaceThreads));
    launch(c, K_SORT, [&] { k_bk_place<D, RT><<<nchp, kPlaceThreads, kTallyWin * sizeof(u32), c->st>>>(stage, n, p.slots, p.g, off, y1, ctrl, si.perm); });
    std::swap(c->y[0], c->y[1]);
    // table 0 from the sorted iterate (runs are contiguous: cheap), then the
    // occupied-slot list of the runs
    enqueue_first_hist<D>(c, p, tabs, n, nb_pts, true);
    launch(c, K_SORT, [&] {
      k_compact<D><<<blocks_for(c, (int64_t)p.slots), kThreads, 0, c->st>>>(tabs[0].ent, p.slots, si.runs, &ctrl->nruns);
    });
    check_launch();
    return true;
  } else {
    launch(c, K_SORT, [&] { k_hist<D, Tab, true><<<nb_pts, kThreads, 0, c->st>>>(y0, n, p.g, tabs[0], ctrl, 0); });
    GS_CUDA(cudaMemcpyAsync(si.runs, tabs[0].list, p.list_cap * sizeof(u32), cudaMemcpyDeviceToDevice, c->st));
    GS_CUDA(cudaMemcpyAsync(&ctrl->nruns, &ctrl->k[0], sizeof(u32), cudaMemcpyDeviceToDevice, c->st));
    launch(c, K_SORT, [&] { k_scan_reduce<D><<<nbs, kThreads, 0, c->st>>>(tabs[0].ent, list, &ctrl->k[0], bsum, p.slots); });
    launch(c, K_SORT, [&] { k_scan_top<<<1, 1024, 0, c->st>>>(bsum, nbs); });
    launch(c, K_SORT, [&] { k_scan_apply<D><<<nbs, kThreads, 0, c->st>>>(tabs[0].ent, list, &ctrl->k[0], bsum, off, p.slots, si.start); });
    double* stage = ensure<double>(c, c->stage, (size_t)n * StageRec<D>::W);
    launch(c, K_SORT, [&] { k_scatter<D, Tab><<<nb_pts, kThreads, 0, c->st>>>(y0, stage, n, p.g, tabs[0], off, si.perm,
                                                                              si.cell0, si.minidx, ctrl); });
    launch(c, K_SORT, [&] { k_unstage<D><<<nb_pts, kThreads, 0, c->st>>>(stage, y1, n, p.g.ld); });
    clear_table<D>(c, p, tabs[0], &ctrl->k[0]);
    check_launch();
    std::swap(c->y[0], c->y[1]);
    return false;
  }
}

struct RunOut {
  int64_t k = 0;
  int iters = 0;
  int converged = 0;
};

template <int D>
RunOut run_engine_d(gs_ctx* c, const Input& in, int64_t n, double h, double eta, int max_iters,
                    int64_t* labels_dev, double* movement_out) {
  // a cell0 copy of an earlier (failed) call may still read the buffer
  if (c->copy) GS_CUDA(cudaStreamWaitEvent(c->st, c->ev_cell0, 0));
  c->cell0_dev = nullptr;
  c->cell0_pending = false;
  c->labels_on_host = false;
  double* y0 = ensure<double>(c, c->y[0], (size_t)soa_ld(n) * D);
  ensure<double>(c, c->y[1], (size_t)soa_ld(n) * D);
  ensure<Ctrl>(c, c->ctrl, 1);
  // sorted dense runs read host-layout rows straight into the sort: the
  // statistics pass then does not materialise the fp64 iterate
  const bool sorted = n >= kSortMinPoints;
  const bool aos_in = in.kind == IN_F64 || in.kind == IN_F32;
  const InitStats s = run_init<D>(c, in, n, h, (sorted && aos_in) ? nullptr : y0);
  Plan p = make_plan(n, D, h, s);
  if (sorted && aos_in && !p.dense) run_init<D>(c, in, n, h, y0);   // hash path sorts the fp64 iterate
  Tabs<D> tabs = make_tabs<D>(c, p);
  ensure<Rec<D>>(c, c->targets, 2 * p.slots);
  const int nb_pts = blocks_for(c, n);
  const int nb_cells = blocks_for(c, (int64_t)p.list_cap);
  ensure<u64>(c, c->partials, 2 * std::max<size_t>((size_t)nb_pts, (size_t)c->sms * 128) + 2);
  ensure<double>(c, c->mv_hist, (size_t)max_iters);
  GS_CUDA(cudaMemsetAsync(ensure<u64>(c, c->wr_hist, (size_t)max_iters), 0, sizeof(u64) * max_iters, c->st));
  u64* fp = ensure<u64>(c, c->fp_hist, (size_t)max_iters);
  ensure<u32>(c, c->k_hist, (size_t)max_iters);
  GS_CUDA(cudaMemsetAsync(fp, 0, sizeof(u64) * max_iters, c->st));
  GS_CUDA(cudaMemsetAsync(c->k_hist.p, 0, sizeof(u32) * max_iters, c->st));
  reset_ctrl(c);
  SortInfo sinfo;
  bool table0 = false;   // the sort already built the table of y_0
  const SrcSoA<D> soa{y0, soa_ld(n)};
  if (sorted && !p.dense)
    table0 = spatial_sort<D>(c, p, tabs.hs, n, sinfo, soa);
  else if (sorted && in.kind == IN_F32)
    table0 = spatial_sort<D>(c, p, tabs.dn, n, sinfo, SrcAoS<D, float>{static_cast<const float*>(in.dev)});
  else if (sorted && in.kind == IN_F64)
    table0 = spatial_sort<D>(c, p, tabs.dn, n, sinfo, SrcAoS<D, double>{static_cast<const double*>(in.dev)});
  else if (sorted)
    table0 = spatial_sort<D>(c, p, tabs.dn, n, sinfo, soa);
  if (sorted && p.dense && c->host_labels) cell0_mark(c, sinfo.cell0, n);
  if (sorted && !p.dense) {
    // k never grows (k_{t+1} <= k_t: y_{t+1} takes at most k_t distinct
    // values), so the loop's hash tables only need 2*k_0 slots: compact
    // tables keep the 3^d probes in L2.  The buffers are clean, only the
    // mask shrinks.
    read_ctrl(c);
    uint64_t cap = 256;
    while (cap < 2ull * c->h_ctrl->nruns) cap <<= 1;
    if (cap < p.slots) {
      p.slots = cap;
      p.g.mask = cap - 1;
      tabs = make_tabs<D>(c, p);
    }
  }
  if (table0)
    ;
  else if (p.dense)
    enqueue_first_hist<D>(c, p, tabs.dn, n, nb_pts, sorted);
  else
    enqueue_first_hist<D>(c, p, tabs.hs, n, nb_pts, sorted, sorted ? &sinfo : nullptr);
  // reference-order sums (default): the first table's sums in np.bincount
  // order, from the input values in original point order
  if (!c->exact_sums) {
    rs_alloc(c, p, D, n, sorted ? sinfo.slots0 : p.slots, p.list_cap, max_iters, c->seq_model);
    InVal<D> V{nullptr, 2, soa_ld(n)};
    if (sorted && aos_in && p.dense)
      V = InVal<D>{in.dev, in.kind == IN_F32 ? 1 : 0, 0};
    else
      V.p = sorted ? c->y[1].p : c->y[0].p;   // the fp64 iterate before the sort's swap
    const double* ys = static_cast<const double*>(c->y[0].p);
    if (p.dense)
      rs_first<D>(c, p, tabs.dn, n, sorted ? &sinfo : nullptr, ys, V, s);
    else
      rs_first<D>(c, p, tabs.hs, n, sorted ? &sinfo : nullptr, ys, V, s);
  }
  // collapsed mode: after iteration 0 the runs of the spatial
  // sort hold one position each; later iterations move runs, not points
  const bool collapsed = c->collapsed && sorted && max_iters > 1;
  if (collapsed) {
    sinfo.rld = (int64_t)((p.list_cap + 127) & ~uint64_t(127));
    sinfo.runpos = ensure<double>(c, c->runposb, (size_t)sinfo.rld * D);
    sinfo.runcnt = ensure<u32>(c, c->runcntb, p.list_cap);
  }
  // device-driven loop: chunks of 4, 8, 16, 32 iterations.  Chunk j+1 is
  // enqueued before the host waits for chunk j's stop flag (a pinned Ctrl
  // snapshot taken right after chunk j), so the device never idles on the
  // host; kernels of iterations past the stop exit on the stamped `done`.
  if (!c->h_snap) {
    GS_CUDA(cudaMallocHost(&c->h_snap, 2 * sizeof(Ctrl)));
    for (cudaEvent_t* e : {&c->ev_snap[0], &c->ev_snap[1]})
      GS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  auto enqueue_chunk = [&](int t0, int m) {
    for (int t = t0; t < t0 + m; ++t) {
      if (collapsed && t >= 1) {
        if (p.dense)
          enqueue_run_iteration<D>(c, p, tabs.dn, t, eta, sinfo, nb_cells);
        else
          enqueue_run_iteration<D>(c, p, tabs.hs, t, eta, sinfo, nb_cells);
        continue;
      }
      if (p.dense)
        enqueue_iteration<D>(c, p, tabs.dn, t, eta, n, nb_pts, nb_cells, nullptr, true, !collapsed);
      else
        enqueue_iteration<D>(c, p, tabs.hs, t, eta, n, nb_pts, nb_cells);
      if (collapsed && t == 0) {
        Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
        const double* y1 = static_cast<const double*>(c->y[0].p);   // y_1, shifted in place
        launch(c, K_SHIFT, [&] {
          k_runs_gather<D><<<nb_cells, kThreads, 0, c->st>>>(y1, p.g.ld, sinfo.runs, &ctrl->nruns, sinfo.start,
                                                              sinfo.end, sinfo.runpos, sinfo.runcnt, sinfo.rld);
        });
      }
    }
    side_join(c);
    check_launch();
  };
  auto snapshot = [&](int slot) {
    GS_CUDA(cudaMemcpyAsync(c->h_snap + slot, c->ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaEventRecord(c->ev_snap[slot], c->st));
  };
  // (the first three chunks are not run ahead: short converging runs would
  // otherwise pay for a chunk of early-exiting launches)
  int t = std::min(4, max_iters), chunk = 4, slot = 0;
  enqueue_chunk(0, t);
  snapshot(0);
  while (true) {
    if (t < 28 && t < max_iters) {   // synchronous chunk boundary (chunks of 4, 8, 16)
      GS_CUDA(cudaEventSynchronize(c->ev_snap[slot]));
      check_flags(c->h_snap[slot].error);
      if (c->h_snap[slot].done) break;
      chunk = std::min(chunk * 2, 32);
      const int m = std::min(chunk, max_iters - t);
      enqueue_chunk(t, m);
      t += m;
      snapshot(slot);
      continue;
    }
    const bool more = t < max_iters;
    if (more) {
      chunk = std::min(chunk * 2, 32);
      const int m = std::min(chunk, max_iters - t);
      enqueue_chunk(t, m);
      t += m;
      snapshot(slot ^ 1);
      cell0_copy_start(c);
    }
    GS_CUDA(cudaEventSynchronize(c->ev_snap[slot]));
    check_flags(c->h_snap[slot].error);
    if (c->h_snap[slot].done || !more) break;
    slot ^= 1;
  }
  cell0_copy_start(c);
  read_ctrl(c);   // everything enqueued has finished; final stop state
  check_flags(c->h_ctrl->error);
  RunOut r;
  r.iters = c->h_ctrl->iters;
  r.converged = c->h_ctrl->done != 0;
  const int e = r.iters & 1;
  const double* yf = static_cast<const double*>(c->y[0].p);   // in-place iterate
  const SortInfo* sp = (sorted && r.iters >= 1) ? &sinfo : nullptr;
  if (p.dense)
    run_extract<D>(c, p, tabs.dn, yf, n, e, labels_dev, sp, true);
  else
    run_extract<D>(c, p, tabs.hs, yf, n, e, labels_dev, sp, true);
  r.k = c->k_last;
  if (movement_out)
    GS_CUDA(cudaMemcpyAsync(movement_out, c->mv_hist.p, sizeof(double) * r.iters, cudaMemcpyDeviceToHost, c->st));
  c->iter_k.assign(r.iters, 0);
  c->iter_fp.assign(r.iters, 0);
  std::vector<u32> kk(r.iters + 1);
  GS_CUDA(cudaMemcpyAsync(kk.data(), c->k_hist.p, sizeof(u32) * r.iters, cudaMemcpyDeviceToHost, c->st));
  GS_CUDA(cudaMemcpyAsync(c->iter_fp.data(), c->fp_hist.p, sizeof(u64) * r.iters, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  for (int i = 0; i < r.iters; ++i) c->iter_k[i] = kk[i];
  c->rsr.on = false;
  c->it_n = n;
  c->it_d = D;
  c->it_sorted = sorted;
  c->it_valid = !collapsed;
  return r;
}

RunOut run_engine(gs_ctx* c, const Input& in, int64_t n, int d, double h, double eta, int max_iters,
                  int64_t* labels_dev, double* movement_out) {
  switch (d) {
#define GS_CASE(DD) \
  case DD:          \
    return run_engine_d<DD>(c, in, n, h, eta, max_iters, labels_dev, movement_out);
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6) GS_CASE(7) GS_CASE(8)
#undef GS_CASE
  }
  fail(GS_EUNSUPPORTED, "unsupported d");
}

void validate_run(int64_t n, int d, double h, double eta, int max_iters) {
  validate_common(n, d, h);
  if (!(std::isfinite(eta) && eta > 0)) fail(GS_EINVAL, "eta must be positive and finite");
  if (max_iters < 1) fail(GS_EINVAL, "max_iters must be a positive integer");
}

// --------------------------------------------------------------- step / tables

template <int D>
void run_step_d(gs_ctx* c, const double* xdev, int64_t n, double h, double* y_out_host, double* movement) {
  double* y0 = ensure<double>(c, c->y[0], (size_t)soa_ld(n) * D);
  ensure<double>(c, c->y[1], (size_t)soa_ld(n) * D);
  ensure<Ctrl>(c, c->ctrl, 1);
  Input in{IN_F64, xdev};
  const InitStats s = run_init<D>(c, in, n, h, y0);
  Plan p = make_plan(n, D, h, s);
  Tabs<D> tabs = make_tabs<D>(c, p);
  ensure<Rec<D>>(c, c->targets, p.slots);
  const int nb_pts = blocks_for(c, n);
  const int nb_cells = blocks_for(c, (int64_t)p.list_cap);
  ensure<u64>(c, c->partials, 2 * std::max<size_t>((size_t)nb_pts, (size_t)c->sms * 128) + 2);
  ensure<double>(c, c->mv_hist, 1);
  GS_CUDA(cudaMemsetAsync(ensure<u64>(c, c->wr_hist, 1), 0, sizeof(u64), c->st));
  GS_CUDA(cudaMemsetAsync(ensure<u64>(c, c->fp_hist, 1), 0, 8, c->st));
  GS_CUDA(cudaMemsetAsync(ensure<u32>(c, c->k_hist, 1), 0, 4, c->st));
  reset_ctrl(c);
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  // reference-order sums: the step equals the reference's bit for bit
  const bool rs = !c->exact_sums;   // (distinct input values: the sequential model is the reference's order too)
  if (rs) rs_alloc(c, p, D, n, p.slots, p.list_cap);
  const InVal<D> V{y0, 2, soa_ld(n)};
  if (p.dense) {
    enqueue_first_hist<D>(c, p, tabs.dn, n, nb_pts);
    if (rs) rs_first<D>(c, p, tabs.dn, n, nullptr, y0, V, s);
    enqueue_iteration<D>(c, p, tabs.dn, 0, -1.0, n, nb_pts, nb_cells);
    clear_table<D>(c, p, tabs.dn[0], &ctrl->k[0]);
    clear_table<D>(c, p, tabs.dn[1], &ctrl->k[1]);
  } else {
    enqueue_first_hist<D>(c, p, tabs.hs, n, nb_pts);
    if (rs) rs_first<D>(c, p, tabs.hs, n, nullptr, y0, V, s);
    enqueue_iteration<D>(c, p, tabs.hs, 0, -1.0, n, nb_pts, nb_cells);
    clear_table<D>(c, p, tabs.hs[0], &ctrl->k[0]);
    clear_table<D>(c, p, tabs.hs[1], &ctrl->k[1]);
  }
  double* aos = ensure<double>(c, c->x_stage, (size_t)n * D);
  launch(c, K_XPOSE, [&] { k_soa_to_aos<D><<<nb_pts, kThreads, 0, c->st>>>(y0, aos, n, p.g.ld); });
  check_launch();
  read_ctrl(c);
  check_flags(c->h_ctrl->error);
  GS_CUDA(cudaMemcpyAsync(y_out_host, aos, sizeof(double) * n * D, cudaMemcpyDeviceToHost, c->st));
  GS_CUDA(cudaMemcpyAsync(movement, c->mv_hist.p, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  sync(c);
}

template <int D, class Tab>
int64_t dump_tables(gs_ctx* c, const Plan& p, Tab* tabs, int64_t cap, int64_t* cells_out, int64_t* counts_out,
                    double* sums_out, int64_t* nc_out, double* ns_out) {
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  read_ctrl(c);
  check_flags(c->h_ctrl->error);
  const int64_t k = c->h_ctrl->k[0];
  if (cap >= k && k > 0) {
    u64* dk = ensure<u64>(c, c->roots, k);
    i64* dc = ensure<i64>(c, c->root_first, k);
    double* ds = ensure<double>(c, c->modes, (size_t)k * D);
    i64* dnc = nullptr;
    double* dns = nullptr;
    if (nc_out) {
      dnc = ensure<i64>(c, c->ranks, k);
      dns = ensure<double>(c, c->aux, (size_t)k * D);
    }
    const double* rs = c->rsr.on ? c->rsr.rs[0] : nullptr;
    launch(c, K_DUMP, [&] { k_dump<D, Tab><<<blocks_for(c, k), kThreads, 0, c->st>>>(p.g, tabs[0], &ctrl->k[0], dk, dc, ds, dnc, dns, rs); });
    check_launch();
    std::vector<u64> hk(k);
    std::vector<i64> hc(k), hnc(nc_out ? k : 0);
    std::vector<double> hsum((size_t)k * D), hns(nc_out ? (size_t)k * D : 0);
    GS_CUDA(cudaMemcpyAsync(hk.data(), dk, k * 8, cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaMemcpyAsync(hc.data(), dc, k * 8, cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaMemcpyAsync(hsum.data(), ds, k * 8 * D, cudaMemcpyDeviceToHost, c->st));
    if (nc_out) {
      GS_CUDA(cudaMemcpyAsync(hnc.data(), dnc, k * 8, cudaMemcpyDeviceToHost, c->st));
      GS_CUDA(cudaMemcpyAsync(hns.data(), dns, k * 8 * D, cudaMemcpyDeviceToHost, c->st));
    }
    sync(c);
    std::vector<int64_t> order(k);
    for (int64_t i = 0; i < k; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return hk[a] < hk[b]; });
    for (int64_t r = 0; r < k; ++r) {
      const int64_t a = order[r];
      for (int j = 0; j < D; ++j) {
        const uint64_t ext = (j == 0) ? (p.g.nkeys / p.g.stride[0]) : (p.g.stride[j - 1] / p.g.stride[j]);
        cells_out[r * D + j] = (int64_t)((hk[a] / p.g.stride[j]) % ext) + p.g.base[j];
        sums_out[r * D + j] = hsum[a * D + j];
        if (nc_out) ns_out[r * D + j] = hns[a * D + j];
      }
      counts_out[r] = hc[a];
      if (nc_out) nc_out[r] = hnc[a];
    }
  }
  launch(c, K_CLEAR, [&] { k_clear<D, Tab><<<blocks_for(c, (int64_t)p.list_cap), kThreads, 0, c->st>>>(tabs[0], &ctrl->k[0]); });
  launch(c, K_CLEAR, [&] { k_reset_count<<<1, 1, 0, c->st>>>(&ctrl->k[0]); });
  check_launch();
  sync(c);
  return k;
}

template <int D>
int64_t run_tables_d(gs_ctx* c, const double* xdev, int64_t n, double h, int64_t cap, int64_t* cells,
                     int64_t* counts, double* sums, int64_t* nc, double* ns) {
  double* y0 = ensure<double>(c, c->y[0], (size_t)soa_ld(n) * D);
  ensure<Ctrl>(c, c->ctrl, 1);
  Input in{IN_F64, xdev};
  const InitStats s = run_init<D>(c, in, n, h, y0);
  Plan p = make_plan(n, D, h, s);
  Tabs<D> tabs = make_tabs<D>(c, p);
  reset_ctrl(c);
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  const int nb_pts = blocks_for(c, n);
  // reference-order sums (default): the reference's tables bit for bit
  const bool rs = !c->exact_sums;   // (distinct input values: the sequential model is the reference's order too)
  if (rs) rs_alloc(c, p, D, n, p.slots, p.list_cap);
  const InVal<D> V{y0, 2, soa_ld(n)};
  if (p.dense) {
    launch(c, K_HIST, [&] { k_hist<D><<<nb_pts, kThreads, 0, c->st>>>(y0, n, p.g, tabs.dn[0], ctrl, 0); });
    if (rs) rs_first<D>(c, p, tabs.dn, n, nullptr, y0, V, s);
    build_list<D>(c, p, tabs.dn[0]);
    return dump_tables<D>(c, p, tabs.dn, cap, cells, counts, sums, nc, ns);
  }
  launch(c, K_HIST, [&] { k_hist<D><<<nb_pts, kThreads, 0, c->st>>>(y0, n, p.g, tabs.hs[0], ctrl, 0); });
  if (rs) rs_first<D>(c, p, tabs.hs, n, nullptr, y0, V, s);
  return dump_tables<D>(c, p, tabs.hs, cap, cells, counts, sums, nc, ns);
}

template <int D>
int64_t run_extract_only_d(gs_ctx* c, const double* xdev, int64_t n, double h, int64_t* labels_dev) {
  double* y0 = ensure<double>(c, c->y[0], (size_t)soa_ld(n) * D);
  ensure<Ctrl>(c, c->ctrl, 1);
  Input in{IN_F64, xdev};
  const InitStats s = run_init<D>(c, in, n, h, y0);
  Plan p = make_plan(n, D, h, s);
  Tabs<D> tabs = make_tabs<D>(c, p);
  reset_ctrl(c);
  if (p.dense)
    run_extract<D>(c, p, tabs.dn, y0, n, 0, labels_dev);
  else
    run_extract<D>(c, p, tabs.hs, y0, n, 0, labels_dev);
  return c->k_last;
}

template <typename F>
int guarded(gs_ctx* c, F&& f) {
  g_err.clear();
  if (!c) {
    g_err = "null context";
    return GS_EINVAL;
  }
  std::lock_guard<std::mutex> lk(c->mu);
  try {
    GS_CUDA(cudaSetDevice(c->device));
    c->st = c->own;
    c->rsr.on = false;   // set by the entry points that use reference-order sums
    f();
    return GS_OK;
  } catch (const Fail& e) {
    // leave the context usable: drain the streams, clean tables next call
    cudaStreamSynchronize(c->st);
    if (c->side) cudaStreamSynchronize(c->side);
    cudaGetLastError();
    c->tables_dirty = true;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    c->tables_dirty = true;
    return GS_ERUNTIME;
  }
}

double* stage_input(gs_ctx* c, const double* x, int64_t n, int d) {
  double* dx = ensure<double>(c, c->x_stage, (size_t)n * d);
  GS_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * n * d, cudaMemcpyHostToDevice, c->st));
  return dx;
}

}  // namespace

// ------------------------------------------------------------- sharded runs
// A row shard of one MeanShift++ run (one process per GPU).  Only the first
// cell table is merged across ranks (integer all-reduce: exact, identical on
// every rank); every later table is derived from the global one (k_derive)
// on every rank alike, so an iteration exchanges just the 4-limb movement.

struct ShardState {
  int d = 0;
  int64_t n = 0;
  int64_t n_total = 0;
  double h = 0;
  int max_iters = 0;
  Plan p{};
  SortInfo si{};
  bool sorted = false;
  bool model = false;      // sequential-model sums (GS_SUMS_SEQMODEL / _REFERENCE contexts); else exact
};

ShardState* shard_of(gs_ctx* c, bool create) {
  if (!c->shard) {
    if (!create) fail(GS_EINVAL, "no sharded run in progress on this context");
    c->shard = new ShardState();
  }
  return c->shard;
}

template <int D>
void shard_plan_d(gs_ctx* c, ShardState* sh, const InitStats& s) {
  Plan p = make_plan(sh->n_total, D, sh->h, s);
  if (!p.dense) fail(GS_EUNSUPPORTED, "row sharding needs a dense lattice table (shard by image instead)");
  p.g.ld = soa_ld(sh->n);
  sh->p = p;
  Tabs<D> tabs = make_tabs<D>(c, p);
  ensure<Rec<D>>(c, c->targets, 2 * p.slots);
  const int nb_pts = blocks_for(c, sh->n);
  ensure<u64>(c, c->partials, 2 * std::max<size_t>((size_t)nb_pts, (size_t)c->sms * 128) + 2);
  ensure<double>(c, c->mv_hist, (size_t)sh->max_iters);
  GS_CUDA(cudaMemsetAsync(ensure<u64>(c, c->wr_hist, (size_t)sh->max_iters), 0, 8 * sh->max_iters, c->st));
  GS_CUDA(cudaMemsetAsync(ensure<u64>(c, c->fp_hist, (size_t)sh->max_iters), 0, 8 * sh->max_iters, c->st));
  GS_CUDA(cudaMemsetAsync(ensure<u32>(c, c->k_hist, (size_t)sh->max_iters), 0, 4 * sh->max_iters, c->st));
  reset_ctrl(c);
  sh->sorted = sh->n >= kSortMinPoints;
  const bool table0 = sh->sorted && spatial_sort<D>(c, p, tabs.dn, sh->n, sh->si,
                                                    SrcSoA<D>{static_cast<const double*>(c->y[0].p), p.g.ld});
  if (!table0) enqueue_first_hist<D>(c, p, tabs.dn, sh->n, nb_pts);
  check_launch();
}

// The merged (global) first table is in buffer 0: with the sequential-model
// sum order its coordinate sums are the exact sums rounded once (as on one
// GPU), for every occupied cell of the GLOBAL table -- later tables are a
// function of the table alone (k_rs_classify, k_rs_runfold), so every rank
// computes the same sums whatever its rows are.
template <int D>
void shard_model_first_d(gs_ctx* c, ShardState* sh) {
  Tabs<D> tabs = make_tabs<D>(c, sh->p);
  RsRun& R = rs_alloc(c, sh->p, D, sh->n, sh->p.slots, sh->p.list_cap, sh->max_iters, true);
  u32* occ = ensure<u32>(c, c->rs_runs, sh->p.list_cap);
  u32* nocc = ensure<u32>(c, c->rs_nocc, 1);
  GS_CUDA(cudaMemsetAsync(nocc, 0, sizeof(u32), c->st));
  launch(c, K_REFSUM, [&] {
    k_compact<D><<<blocks_for(c, (int64_t)sh->p.slots), kThreads, 0, c->st>>>(tabs.dn[0].ent, sh->p.slots, occ, nocc);
  });
  GS_CUDA(cudaMemsetAsync(R.ctl, 0, sizeof(RsCtl), c->st));
  LowBits lb{};
  launch(c, K_REFSUM, [&] {
    k_rs_first<D, DenseTable<D>><<<blocks_for(c, (int64_t)sh->p.list_cap), kThreads, 0, c->st>>>(
        sh->p.g, tabs.dn[0], occ, nocc, nullptr, nullptr, false, false, lb, R.rc[0], R.runkey, R.outslot, R.rs[0],
        R.ctl, R.seglen, R.sstart, R.send, R.seglist, R.runkv, nullptr, nullptr, true);
  });
  check_launch();
}

template <int D>
void shard_iterate_d(gs_ctx* c, ShardState* sh, int t, u64* limbs) {
  Tabs<D> tabs = make_tabs<D>(c, sh->p);
  c->rsr.on = sh->model;   // (entry points clear it)
  enqueue_iteration<D>(c, sh->p, tabs.dn, t, 0.0, sh->n, blocks_for(c, sh->n),
                       blocks_for(c, (int64_t)sh->p.list_cap), limbs, true, true);
  check_launch();
}

template <int D>
void shard_components_d(gs_ctx* c, ShardState* sh, u32 offset, long long* minima) {
  Tabs<D> tabs = make_tabs<D>(c, sh->p);
  side_join(c);
  read_ctrl(c);
  check_flags(c->h_ctrl->error);
  const int e = c->h_ctrl->iters & 1;
  const double* yf = static_cast<const double*>(c->y[0].p);   // in-place iterate
  const SortInfo* sp = (sh->sorted && c->h_ctrl->iters >= 1) ? &sh->si : nullptr;
  extract_components<D>(c, sh->p, tabs.dn, yf, sh->n, e, sp, true, offset);
  GS_CUDA(cudaMemsetAsync(minima, 0x7f, sh->p.slots * sizeof(long long), c->st));
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  launch(c, K_COMP, [&] {
    k_export_minima<D, DenseTable<D>><<<blocks_for(c, (int64_t)sh->p.list_cap), kThreads, 0, c->st>>>(
        tabs.dn[e], &ctrl->k[e], static_cast<u32*>(c->par.p), static_cast<u32*>(c->first.p), minima);
  });
  check_launch();
}

template <int D>
void shard_finish_d(gs_ctx* c, ShardState* sh, const long long* minima, int64_t* labels_dev) {
  Tabs<D> tabs = make_tabs<D>(c, sh->p);
  const int e = c->h_ctrl->iters & 1;
  const double* yf = static_cast<const double*>(c->y[0].p);   // in-place iterate
  Ctrl* ctrl = static_cast<Ctrl*>(c->ctrl.p);
  launch(c, K_COMP, [&] {
    k_import_minima<D, DenseTable<D>><<<blocks_for(c, (int64_t)sh->p.list_cap), kThreads, 0, c->st>>>(
        tabs.dn[e], &ctrl->k[e], static_cast<u32*>(c->par.p), static_cast<u32*>(c->first.p), minima);
  });
  const SortInfo* sp = (sh->sorted && c->h_ctrl->iters >= 1) ? &sh->si : nullptr;
  extract_finish<D>(c, sh->p, tabs.dn, yf, sh->n, e, labels_dev, sp);
}

// GS_ONLY_D (development builds: nvcc -DGS_ONLY_D=3) instantiates one
// dimension only; the shipped library is built without it.
#ifdef GS_ONLY_D
#define GS_DISPATCH(d, CALL)                                                    \
  switch (d) {                                                                  \
    case GS_ONLY_D: { constexpr int DD = GS_ONLY_D; CALL; } break;               \
    default: fail(GS_EUNSUPPORTED, "development build: one dimension only");      \
  }
#else
#define GS_DISPATCH(d, CALL)                                                    \
  switch (d) {                                                                  \
    case 1: { constexpr int DD = 1; CALL; } break;                               \
    case 2: { constexpr int DD = 2; CALL; } break;                               \
    case 3: { constexpr int DD = 3; CALL; } break;                               \
    case 4: { constexpr int DD = 4; CALL; } break;                               \
    case 5: { constexpr int DD = 5; CALL; } break;                               \
    case 6: { constexpr int DD = 6; CALL; } break;                               \
    case 7: { constexpr int DD = 7; CALL; } break;                               \
    case 8: { constexpr int DD = 8; CALL; } break;                               \
    default: fail(GS_EUNSUPPORTED, "unsupported d");                              \
  }
#endif

// ===================================================================== C ABI

extern "C" {

const char* gs_last_error(void) { return g_err.c_str(); }

const char* gs_version(void) { return "gridshift-b200 0.1 sm_100a"; }

int gs_ctx_create(int device, gs_ctx** out) {
  g_err.clear();
  if (!out) return GS_EINVAL;
  *out = nullptr;
  gs_ctx* c = new gs_ctx();
  try {
    c->device = device;
    GS_CUDA(cudaSetDevice(device));
    GS_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
    GS_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->st = c->own;
    GS_CUDA(cudaMallocHost(&c->h_ctrl, sizeof(Ctrl)));
    GS_CUDA(cudaMallocHost(&c->h_stats, sizeof(InitStats)));
    GS_CUDA(cudaMallocHost(&c->h_small, 64));
    ensure<Ctrl>(c, c->ctrl, 1);
    sync(c);
  } catch (const Fail& e) {
    delete c;
    return e.code;
  }
  *out = c;
  return GS_OK;
}

void gs_ctx_destroy(gs_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->own) cudaStreamSynchronize(c->own);
  Buf* bufs[] = {&c->x_stage, &c->y[0], &c->y[1], &c->ent[0], &c->ent[1], &c->keys[0], &c->keys[1],
                 &c->list[0], &c->list[1], &c->targets, &c->partials, &c->par, &c->first, &c->aux,
                 &c->roots, &c->root_first, &c->ranks, &c->modes, &c->labels, &c->mv_hist,
                 &c->fp_hist, &c->k_hist, &c->stats, &c->ctrl, &c->perm, &c->colsum, &c->track,
                 &c->track_out, &c->bitmaps, &c->scan, &c->runoff, &c->runstart, &c->runmin,
                 &c->runlist, &c->cell0, &c->stage, &c->runposb, &c->runcntb, &c->bkcnt, &c->bktot, &c->bocc, &c->bmask, &c->wr_hist};
  for (Buf* b : bufs)
    if (b->p) cudaFree(b->p);
  Buf* rbufs[] = {&c->rsb[0], &c->rsb[1], &c->rs_nsrc, &c->rs_mid, &c->rs_out, &c->rs_rc[0], &c->rs_rc[1],
                  &c->rs_rkey, &c->rs_rval, &c->rs_k[0], &c->rs_k[1], &c->rs_v[0], &c->rs_v[1], &c->rs_cnt,
                  &c->rs_scan, &c->rs_start, &c->rs_end, &c->rs_wsum, &c->rs_wpre, &c->rs_wdelta, &c->rs_ctl,
                  &c->rs_cell0, &c->rs_runs, &c->rs_seglen, &c->rs_segbeg, &c->rs_segcur, &c->rs_seglist,
                  &c->rs_runseg, &c->rs_segscan, &c->rs_runkv, &c->rs_tag[0], &c->rs_tag[1], &c->rs_stats,
                  &c->rs_lowrun, &c->rs_lst[0], &c->rs_lst[1], &c->rs_shead, &c->rs_snext, &c->rs_segdone,
                  &c->rs_atop, &c->rs_ctalist, &c->rs_nocc};
  for (Buf* b : rbufs)
    if (b->p) cudaFree(b->p);
  if (c->h_ctrl) cudaFreeHost(c->h_ctrl);
  if (c->h_stats) cudaFreeHost(c->h_stats);
  if (c->h_small) cudaFreeHost(c->h_small);
  for (cudaEvent_t e : c->prof.pool) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_fork, c->ev_join, c->ev_rec[0], c->ev_rec[1], c->ev_shift[0], c->ev_shift[1],
                        c->ev_snap[0], c->ev_snap[1], c->ev_pace[0], c->ev_pace[1]})
    if (e) cudaEventDestroy(e);
  if (c->h_snap) cudaFreeHost(c->h_snap);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->copy) cudaStreamSynchronize(c->copy);
  if (c->h_cell0) cudaFreeHost(c->h_cell0);
  if (c->h_slotlab) cudaFreeHost(c->h_slotlab);
  if (c->slotlab.p) cudaFree(c->slotlab.p);
  for (cudaEvent_t e : {c->ev_sorted, c->ev_cell0})
    if (e) cudaEventDestroy(e);
  if (c->copy) cudaStreamDestroy(c->copy);
  delete c->shard;
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
}

int gs_meanshiftpp(gs_ctx* c, const double* x, int64_t n, int32_t d, double h, double eta,
                   int32_t max_iters, int64_t* labels_out, int64_t* k_out, int32_t* iters_out,
                   double* movement_out, int32_t* converged_out) {
  return guarded(c, [&] {
    validate_run(n, d, h, eta, max_iters);
    if (!x || !labels_out) fail(GS_EINVAL, "null buffer");
    const double* dx = stage_input(c, x, n, d);
    c->xfer_h2d = (int64_t)sizeof(double) * n * d;
    int64_t* dl = ensure<int64_t>(c, c->labels, n);
    Input in{IN_F64, dx};
    RunOut r;
    {
      HostLabelRequest req(c);
      r = run_engine(c, in, n, d, h, eta, max_iters, dl, movement_out);
    }
    deliver_labels(c, dl, labels_out, n);
    if (k_out) *k_out = r.k;
    if (iters_out) *iters_out = r.iters;
    if (converged_out) *converged_out = r.converged;
  });
}

int gs_meanshiftpp_host(gs_ctx* c, const void* x, int32_t dtype, int64_t n, int32_t d, double h, double eta,
                        int32_t max_iters, int64_t* labels_out, int64_t* k_out, int32_t* iters_out,
                        double* movement_out, int32_t* converged_out) {
  return guarded(c, [&] {
    validate_run(n, d, h, eta, max_iters);
    if (!x || !labels_out) fail(GS_EINVAL, "null buffer");
    if (dtype != GS_DTYPE_F64 && dtype != GS_DTYPE_F32) fail(GS_EINVAL, "dtype must be f64 or f32");
    const size_t esz = dtype == GS_DTYPE_F64 ? 8 : 4;
    unsigned char* dx = ensure<unsigned char>(c, c->x_stage, (size_t)n * d * esz);
    GS_CUDA(cudaMemcpyAsync(dx, x, (size_t)n * d * esz, cudaMemcpyHostToDevice, c->st));
    c->xfer_h2d = (int64_t)(n * d * esz);
    int64_t* dl = ensure<int64_t>(c, c->labels, n);
    Input in{dtype == GS_DTYPE_F64 ? IN_F64 : IN_F32, dx};
    RunOut r;
    {
      HostLabelRequest req(c);
      r = run_engine(c, in, n, d, h, eta, max_iters, dl, movement_out);
    }
    deliver_labels(c, dl, labels_out, n);
    if (k_out) *k_out = r.k;
    if (iters_out) *iters_out = r.iters;
    if (converged_out) *converged_out = r.converged;
  });
}

int gs_meanshiftpp_device(gs_ctx* c, const void* x_dev, int32_t dtype, int64_t n, int32_t d, double h,
                          double eta, int32_t max_iters, int64_t* labels_dev, int64_t* k_out,
                          int32_t* iters_out, double* movement_out, int32_t* converged_out, void* stream) {
  return guarded(c, [&] {
    validate_run(n, d, h, eta, max_iters);
    if (!x_dev || !labels_dev) fail(GS_EINVAL, "null buffer");
    if (dtype != GS_DTYPE_F64 && dtype != GS_DTYPE_F32) fail(GS_EINVAL, "dtype must be f64 or f32");
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    Input in{dtype == GS_DTYPE_F64 ? IN_F64 : IN_F32, x_dev};
    RunOut r = run_engine(c, in, n, d, h, eta, max_iters, labels_dev, movement_out);
    sync(c);
    if (k_out) *k_out = r.k;
    if (iters_out) *iters_out = r.iters;
    if (converged_out) *converged_out = r.converged;
  });
}

int gs_segment_image(gs_ctx* c, const uint8_t* pixels, int32_t height, int32_t width, int32_t mode,
                     double scale, double h, double eta, int32_t max_iters, int64_t* labels_out,
                     int64_t* k_out, int32_t* iters_out, double* movement_out, int32_t* converged_out) {
  return guarded(c, [&] {
    if (height < 1 || width < 1) fail(GS_EINVAL, "image must contain at least one pixel");
    if (mode != 0 && mode != 1) fail(GS_EINVAL, "mode must be one of ('rgb', 'rgbxy')");
    const int64_t n = (int64_t)height * width;
    const int d = mode == 0 ? 3 : 5;
    validate_run(n, d, h, eta, max_iters);
    if (!std::isfinite(scale)) fail(GS_EINVAL, "point data contains NaN or infinite entries");
    unsigned char* dp = ensure<unsigned char>(c, c->x_stage, (size_t)n * 3);
    GS_CUDA(cudaMemcpyAsync(dp, pixels, (size_t)n * 3, cudaMemcpyHostToDevice, c->st));
    c->xfer_h2d = n * 3;
    int64_t* dl = ensure<int64_t>(c, c->labels, n);
    Input in{IN_IMAGE, dp, width, scale};
    RunOut r;
    {
      HostLabelRequest req(c);
      r = run_engine(c, in, n, d, h, eta, max_iters, dl, movement_out);
    }
    // per-segment colour sums on device while the labels travel
    u64* cs = ensure<u64>(c, c->colsum, (size_t)r.k * 4);
    GS_CUDA(cudaMemsetAsync(cs, 0, sizeof(u64) * 4 * (size_t)r.k, c->st));
    const bool by_cell = c->labels_on_host;
    launch(c, K_LABELS, [&] {
      k_label_colors<<<blocks_for(c, n), kThreads, 0, c->st>>>(dp, n, by_cell ? c->cell0_dev : nullptr,
                                                              by_cell ? static_cast<const u32*>(c->slotlab.p) : nullptr,
                                                              reinterpret_cast<const i64*>(dl), cs);
    });
    std::vector<u64> hs((size_t)r.k * 4);
    GS_CUDA(cudaMemcpyAsync(hs.data(), cs, sizeof(u64) * hs.size(), cudaMemcpyDeviceToHost, c->st));
    deliver_labels(c, dl, labels_out, n);   // synchronises the stream
    c->xfer_d2h += (int64_t)(sizeof(u64) * hs.size());
    c->colors_host.resize((size_t)r.k * 3);
    for (int64_t q = 0; q < r.k; ++q)
      for (int ch = 0; ch < 3; ++ch)
        c->colors_host[q * 3 + ch] = (double)hs[q * 4 + ch] / (double)hs[q * 4 + 3];
    if (k_out) *k_out = r.k;
    if (iters_out) *iters_out = r.iters;
    if (converged_out) *converged_out = r.converged;
  });
}

int gs_fetch_mean_colors(gs_ctx* c, double* colors_out, int64_t cap_rows) {
  return guarded(c, [&] {
    if (c->colors_host.empty()) fail(GS_EINVAL, "no segmentation on this context yet");
    if (cap_rows * 3 < (int64_t)c->colors_host.size()) fail(GS_EINVAL, "mean colour buffer too small");
    memcpy(colors_out, c->colors_host.data(), sizeof(double) * c->colors_host.size());
  });
}

int gs_ctx_set_option(gs_ctx* c, int32_t option, int64_t value) {
  return guarded(c, [&] {
    if (option == GS_OPT_COLLAPSED)
      c->collapsed = value != 0;
    else if (option == GS_OPT_SUMS && (value == GS_SUMS_REFERENCE || value == GS_SUMS_EXACT || value == GS_SUMS_SEQMODEL))
    {
      c->exact_sums = value == GS_SUMS_EXACT;
      c->seq_model = value == GS_SUMS_SEQMODEL;
    }
    else
      fail(GS_EINVAL, "unknown option or value");
  });
}

int gs_fetch_modes(gs_ctx* c, double* modes_out, int64_t cap_rows) {
  return guarded(c, [&] {
    if (cap_rows < c->k_last) fail(GS_EINVAL, "modes buffer too small");
    memcpy(modes_out, c->modes_host.data(), sizeof(double) * c->modes_host.size());
  });
}

int gs_profile(gs_ctx* c, int32_t mode, double* ms_out, int64_t* launches_out, int32_t cap) {
  return guarded(c, [&] {
    if (mode == 1 || mode == 0) {  // enable / disable, resetting the counters
      c->prof.on = (mode == 1);
      c->prof.used = 0;
      c->prof.rec.clear();
      for (auto& l : c->prof.launches) l = 0;
      return;
    }
    // mode 2: fetch accumulated per-kind device time (ms) and launch counts
    sync(c);
    double ms[K_NKINDS] = {};
    for (auto& r : c->prof.rec) {
      float t = 0.f;
      GS_CUDA(cudaEventElapsedTime(&t, c->prof.pool[r.second], c->prof.pool[r.second + 1]));
      ms[r.first] += t;
    }
    for (int k = 0; k < K_NKINDS && k < cap; ++k) {
      if (ms_out) ms_out[k] = ms[k];
      if (launches_out) launches_out[k] = c->prof.launches[k];
    }
  });
}

const char* gs_profile_kind(int32_t kind) {
  return (kind >= 0 && kind < K_NKINDS) ? kKindNames[kind] : "";
}

int gs_fetch_trace(gs_ctx* c, int64_t* k_per_iter, uint64_t* fp_per_iter, int32_t cap) {
  return guarded(c, [&] {
    const int m = std::min<int>(cap, (int)c->iter_k.size());
    for (int i = 0; i < m; ++i) {
      if (k_per_iter) k_per_iter[i] = c->iter_k[i];
      if (fp_per_iter) fp_per_iter[i] = c->iter_fp[i];
    }
  });
}

int gs_fetch_refsum_stats(gs_ctx* c, uint32_t* out, int32_t rows) {
  return guarded(c, [&] {
    if (!c->rsr.stats || rows > c->rsr.stats_rows) fail(GS_EINVAL, "no reference-order statistics of that size");
    GS_CUDA(cudaMemcpyAsync(out, c->rsr.stats, 20ull * rows, cudaMemcpyDeviceToHost, c->st));
    sync(c);
  });
}

int gs_fetch_iterate(gs_ctx* c, double* y_out, int64_t n) {
  return guarded(c, [&] {
    if (!c->it_valid || n != c->it_n || !y_out)
      fail(GS_EINVAL, "no per-point iterate of that size from the last run on this context");
    const int d = c->it_d;
    double* out = ensure<double>(c, c->x_stage, (size_t)n * d);
    const double* y = static_cast<const double*>(c->y[0].p);
    const u32* cell0 = c->it_sorted ? static_cast<const u32*>(c->cell0.p) : nullptr;
    const u32* start = c->it_sorted ? static_cast<const u32*>(c->runstart.p) : nullptr;
    launch(c, K_XPOSE, [&] {
      k_iterate_out<<<blocks_for(c, n), kThreads, 0, c->st>>>(y, soa_ld(n), d, cell0, start, n, out);
    });
    check_launch();
    GS_CUDA(cudaMemcpyAsync(y_out, out, sizeof(double) * n * d, cudaMemcpyDeviceToHost, c->st));
    sync(c);
  });
}

int gs_fetch_shift_bytes(gs_ctx* c, uint64_t* bytes_per_iter, int32_t cap) {
  return guarded(c, [&] {
    const int m = std::min<int>(cap, c->h_ctrl ? c->h_ctrl->iters : 0);
    if (m > 0 && c->wr_hist.p) {
      GS_CUDA(cudaMemcpyAsync(bytes_per_iter, c->wr_hist.p, sizeof(uint64_t) * m, cudaMemcpyDeviceToHost, c->st));
      sync(c);
    }
  });
}

int gs_fetch_transfer_bytes(gs_ctx* c, int64_t* h2d_bytes, int64_t* d2h_bytes) {
  return guarded(c, [&] {
    if (h2d_bytes) *h2d_bytes = c->xfer_h2d;
    if (d2h_bytes) *d2h_bytes = c->xfer_d2h;
  });
}

int gs_shift_step(gs_ctx* c, const double* y, int64_t n, int32_t d, double h, double* y_out,
                  double* movement_out) {
  return guarded(c, [&] {
    validate_common(n, d, h);
    const double* dx = stage_input(c, y, n, d);
    switch (d) {
#define GS_CASE(DD) \
  case DD:          \
    run_step_d<DD>(c, dx, n, h, y_out, movement_out); \
    break;
      GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6) GS_CASE(7) GS_CASE(8)
#undef GS_CASE
    }
  });
}

int gs_build_tables(gs_ctx* c, const double* y, int64_t n, int32_t d, double h, int64_t cap,
                    int64_t* cells_out, int64_t* counts_out, double* sums_out, int64_t* nbr_counts_out,
                    double* nbr_sums_out, int64_t* k_out) {
  return guarded(c, [&] {
    validate_common(n, d, h);
    const double* dx = stage_input(c, y, n, d);
    int64_t k = 0;
    switch (d) {
#define GS_CASE(DD) \
  case DD:          \
    k = run_tables_d<DD>(c, dx, n, h, cap, cells_out, counts_out, sums_out, nbr_counts_out, nbr_sums_out); \
    break;
      GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6) GS_CASE(7) GS_CASE(8)
#undef GS_CASE
    }
    if (k_out) *k_out = k;
  });
}

int gs_extract_clusters(gs_ctx* c, const double* y, int64_t n, int32_t d, double h, int64_t* labels_out,
                        int64_t* k_out) {
  return guarded(c, [&] {
    validate_common(n, d, h);
    const double* dx = stage_input(c, y, n, d);
    int64_t* dl = ensure<int64_t>(c, c->labels, n);
    int64_t k = 0;
    switch (d) {
#define GS_CASE(DD) \
  case DD:          \
    k = run_extract_only_d<DD>(c, dx, n, h, dl); \
    break;
      GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6) GS_CASE(7) GS_CASE(8)
#undef GS_CASE
    }
    GS_CUDA(cudaMemcpyAsync(labels_out, dl, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    if (k_out) *k_out = k;
  });
}

int gs_track_sequence(gs_ctx* c, const uint8_t* frames, int32_t n_frames, int32_t height, int32_t width,
                      double cx, double cy, int32_t w, int32_t h_px, const int64_t* bins, int32_t nb,
                      double h, int32_t update_bins, int32_t init_matches, double tol, int32_t max_iters,
                      double* cx_out, double* cy_out, int32_t* lost_out, int64_t* matches_out,
                      int64_t* nbins_out, uint32_t* bitmap_hist_out) {
  return guarded(c, [&] {
    if (!(std::isfinite(h) && h > 0.0)) fail(GS_EINVAL, "bandwidth must be a positive finite real");
    if (n_frames < 1 || height < 1 || width < 1) fail(GS_EINVAL, "need at least one non-empty frame");
    if (w < 1 || h_px < 1) fail(GS_EINVAL, "window extents must be positive");
    if (nb < 1) fail(GS_EINVAL, "bin set cannot be empty");
    if (max_iters < 1) fail(GS_EINVAL, "max_iters must be positive");
    const double Ld = std::floor(255.0 / h) + 1.0;
    if (Ld > 645.0) fail(GS_EUNSUPPORTED, "colour bandwidth too small for the bitmap bin set");
    const int L = (int)Ld;
    const int64_t cells = (int64_t)L * L * L;
    const int words = (int)((cells + 31) / 32);
    std::vector<u32> bm(words, 0u);
    for (int i = 0; i < nb; ++i) {
      const int64_t a = bins[3 * i], b = bins[3 * i + 1], cc = bins[3 * i + 2];
      if (a < 0 || b < 0 || cc < 0 || a >= L || b >= L || cc >= L)
        fail(GS_EINVAL, "bin set holds a colour cell outside [0, floor(255/h)]^3");
      const int64_t code = (a * L + b) * L + cc;
      bm[code >> 5] |= 1u << (code & 31);
    }
    int lut[256];
    for (int v = 0; v < 256; ++v) lut[v] = (int)std::floor((double)v / h);
    const size_t fbytes = (size_t)n_frames * height * width * 3;
    unsigned char* df = ensure<unsigned char>(c, c->track, fbytes);
    GS_CUDA(cudaMemcpyAsync(df, frames, fbytes, cudaMemcpyHostToDevice, c->st));
    u32* dbm = ensure<u32>(c, c->bitmaps, (2 + (size_t)n_frames) * words + 256);
    int* dlut = reinterpret_cast<int*>(dbm + 2 * words);
    u32* dhist = dbm + 2 * words + 256;
    GS_CUDA(cudaMemcpyAsync(dhist, bm.data(), words * sizeof(u32), cudaMemcpyHostToDevice, c->st));
    GS_CUDA(cudaMemcpyAsync(dbm, bm.data(), words * sizeof(u32), cudaMemcpyHostToDevice, c->st));
    GS_CUDA(cudaMemcpyAsync(dlut, lut, sizeof lut, cudaMemcpyHostToDevice, c->st));
    const size_t T = (size_t)n_frames;
    char* o = ensure<char>(c, c->track_out, T * (8 + 8 + 4 + 8 + 8) + 64);
    double* dcx = reinterpret_cast<double*>(o);
    double* dcy = dcx + T;
    long long* dm = reinterpret_cast<long long*>(dcy + T);
    long long* dnb = dm + T;
    int* dlost = reinterpret_cast<int*>(dnb + T);
    // row 0 = the init state (track.py:199-200)
    const double r0[2] = {cx, cy};
    const long long m0[2] = {init_matches, nb};
    const int l0 = 0;
    GS_CUDA(cudaMemcpyAsync(dcx, &r0[0], 8, cudaMemcpyHostToDevice, c->st));
    GS_CUDA(cudaMemcpyAsync(dcy, &r0[1], 8, cudaMemcpyHostToDevice, c->st));
    GS_CUDA(cudaMemcpyAsync(dm, &m0[0], 8, cudaMemcpyHostToDevice, c->st));
    GS_CUDA(cudaMemcpyAsync(dnb, &m0[1], 8, cudaMemcpyHostToDevice, c->st));
    GS_CUDA(cudaMemcpyAsync(dlost, &l0, 4, cudaMemcpyHostToDevice, c->st));
    TrackParams tp{};
    tp.n_frames = n_frames;
    tp.height = height;
    tp.width = width;
    tp.w = w;
    tp.hp = h_px;
    tp.L = L;
    tp.update_bins = update_bins ? 1 : 0;
    tp.max_iters = max_iters;
    tp.tol = tol;
    tp.cx0 = cx;
    tp.cy0 = cy;
    tp.words = words;
    tp.init_matches = init_matches;
    launch(c, K_TRACK, [&] { k_track<<<1, kTrackThreads, 0, c->st>>>(df, tp, dlut, dbm, dbm + words, dcx, dcy, dlost, dm, dnb,
                                            dhist); });
    check_launch();
    GS_CUDA(cudaMemcpyAsync(cx_out, dcx, 8 * T, cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaMemcpyAsync(cy_out, dcy, 8 * T, cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaMemcpyAsync(matches_out, dm, 8 * T, cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaMemcpyAsync(nbins_out, dnb, 8 * T, cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaMemcpyAsync(lost_out, dlost, 4 * T, cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaMemcpyAsync(bm.data(), dbm, words * sizeof(u32), cudaMemcpyDeviceToHost, c->st));
    if (bitmap_hist_out)
      GS_CUDA(cudaMemcpyAsync(bitmap_hist_out, dhist, T * words * sizeof(u32), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    c->track_bins.clear();
    for (int64_t code = 0; code < cells; ++code)
      if ((bm[code >> 5] >> (code & 31)) & 1u) {
        c->track_bins.push_back(code / ((int64_t)L * L));
        c->track_bins.push_back((code / L) % L);
        c->track_bins.push_back(code % L);
      }
  });
}

int gs_fetch_track_bins(gs_ctx* c, int64_t* bins_out, int32_t cap, int32_t* nb_out) {
  return guarded(c, [&] {
    const int32_t nb = (int32_t)(c->track_bins.size() / 3);
    if (nb_out) *nb_out = nb;
    if (bins_out && cap >= nb) memcpy(bins_out, c->track_bins.data(), c->track_bins.size() * 8);
  });
}

int gs_shard_init(gs_ctx* c, const void* x_dev, int32_t dtype, int64_t n_local, int32_t d, double h,
                  void* stream, int64_t* cmin_out, int64_t* cmax_out, double* absmax_out, int32_t* flags_out) {
  return guarded(c, [&] {
    validate_common(n_local, d, h);
    if (!x_dev) fail(GS_EINVAL, "null buffer");
    if (dtype != GS_DTYPE_F64 && dtype != GS_DTYPE_F32) fail(GS_EINVAL, "dtype must be f64 or f32");
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    ShardState* sh = shard_of(c, true);
    sh->d = d;
    sh->n = n_local;
    sh->h = h;
    Input in{dtype == GS_DTYPE_F64 ? IN_F64 : IN_F32, x_dev};
    InitStats st{};
    GS_DISPATCH(d, {
      double* y0 = ensure<double>(c, c->y[0], (size_t)soa_ld(n_local) * DD);
      ensure<double>(c, c->y[1], (size_t)soa_ld(n_local) * DD);
      ensure<Ctrl>(c, c->ctrl, 1);
      st = run_init<DD>(c, in, n_local, h, y0);
    });
    for (int j = 0; j < d; ++j) {
      cmin_out[j] = st.cmin[j];
      cmax_out[j] = st.cmax[j];
      memcpy(&absmax_out[j], &st.absmax[j], 8);
    }
    *flags_out = st.flags;
  });
}

int gs_shard_plan(gs_ctx* c, const int64_t* cmin, const int64_t* cmax, const double* absmax, int32_t flags,
                  int64_t n_total, int32_t max_iters, void* stream, int64_t* table_words_out) {
  return guarded(c, [&] {
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    ShardState* sh = shard_of(c, false);
    if (max_iters < 1) fail(GS_EINVAL, "max_iters must be a positive integer");
    if (n_total < sh->n || n_total >= (int64_t)UINT32_MAX) fail(GS_EINVAL, "bad n_total");
    sh->n_total = n_total;
    sh->max_iters = max_iters;
    InitStats s{};
    for (int j = 0; j < sh->d; ++j) {
      s.cmin[j] = cmin[j];
      s.cmax[j] = cmax[j];
      memcpy(&s.absmax[j], &absmax[j], 8);
    }
    s.flags = flags;
    GS_DISPATCH(sh->d, shard_plan_d<DD>(c, sh, s));
    *table_words_out = (int64_t)sh->p.slots * (1 + 2 * sh->d);
  });
}

int gs_shard_table_io(gs_ctx* c, void* buf_dev, int32_t to_device_table, void* stream) {
  return guarded(c, [&] {
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    ShardState* sh = shard_of(c, false);
    const size_t bytes = sh->p.slots * 8 * (1 + 2 * (size_t)sh->d);
    if (to_device_table) {
      GS_CUDA(cudaMemcpyAsync(c->ent[0].p, buf_dev, bytes, cudaMemcpyDeviceToDevice, c->st));
      sh->model = !c->exact_sums;
      if (sh->model) GS_DISPATCH(sh->d, shard_model_first_d<DD>(c, sh));
    } else
      GS_CUDA(cudaMemcpyAsync(buf_dev, c->ent[0].p, bytes, cudaMemcpyDeviceToDevice, c->st));
  });
}

int gs_shard_iterate(gs_ctx* c, int32_t t, void* limbs_dev, void* stream) {
  return guarded(c, [&] {
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    ShardState* sh = shard_of(c, false);
    if (t < 0 || t >= sh->max_iters) fail(GS_EINVAL, "iteration out of range");
    GS_DISPATCH(sh->d, shard_iterate_d<DD>(c, sh, t, static_cast<u64*>(limbs_dev)));
  });
}

int gs_shard_converge(gs_ctx* c, int32_t t, const void* limbs_dev, double eta, void* stream) {
  return guarded(c, [&] {
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    ShardState* sh = shard_of(c, false);
    launch(c, K_SHIFT, [&] {
      k_converge<<<1, 1, 0, c->st>>>(static_cast<const u64*>(limbs_dev), sh->p.g, static_cast<Ctrl*>(c->ctrl.p),
                                     static_cast<double*>(c->mv_hist.p), t, eta);
    });
    if (c->side) GS_CUDA(cudaEventRecord(c->ev_shift[t & 1], c->st));   // see enqueue_iteration
    check_launch();
  });
}

int gs_shard_status(gs_ctx* c, int32_t* done_out, int32_t* iters_out, void* stream) {
  return guarded(c, [&] {
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    shard_of(c, false);
    side_join(c);   // the table chain may run ahead on the side stream
    read_ctrl(c);
    check_flags(c->h_ctrl->error);
    *done_out = c->h_ctrl->done != 0;
    *iters_out = c->h_ctrl->iters;
  });
}

int gs_shard_components(gs_ctx* c, int64_t global_offset, void* minima_dev, void* stream, int64_t* slots_out) {
  return guarded(c, [&] {
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    ShardState* sh = shard_of(c, false);
    GS_DISPATCH(sh->d, shard_components_d<DD>(c, sh, (u32)global_offset, static_cast<long long*>(minima_dev)));
    *slots_out = (int64_t)sh->p.slots;
  });
}

int gs_shard_finish(gs_ctx* c, const void* minima_dev, int64_t* labels_dev, void* stream, int64_t* k_out,
                    int32_t* iters_out, double* movement_out, int32_t* converged_out) {
  return guarded(c, [&] {
    c->st = static_cast<cudaStream_t>(stream);   // NULL = legacy default stream
    ShardState* sh = shard_of(c, false);
    GS_DISPATCH(sh->d, shard_finish_d<DD>(c, sh, static_cast<const long long*>(minima_dev), labels_dev));
    const int iters = c->h_ctrl->iters;
    if (movement_out)
      GS_CUDA(cudaMemcpyAsync(movement_out, c->mv_hist.p, sizeof(double) * iters, cudaMemcpyDeviceToHost, c->st));
    c->iter_k.assign(iters, 0);
    c->iter_fp.assign(iters, 0);
    std::vector<u32> kk(iters + 1);
    GS_CUDA(cudaMemcpyAsync(kk.data(), c->k_hist.p, sizeof(u32) * iters, cudaMemcpyDeviceToHost, c->st));
    GS_CUDA(cudaMemcpyAsync(c->iter_fp.data(), c->fp_hist.p, sizeof(u64) * iters, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    for (int i = 0; i < iters; ++i) c->iter_k[i] = kk[i];
    *k_out = c->k_last;
    *iters_out = iters;
    *converged_out = c->h_ctrl->done != 0;
    delete c->shard;
    c->shard = nullptr;
  });
}

}  // extern "C"
