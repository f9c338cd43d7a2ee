// gridshift-b200: reference-order cell sums (the default numerics).
//
// The reference builds every per-cell coordinate sum with np.bincount, i.e.
// sequentially in fp64, in point (index) order, starting from 0.0
// (grid.py:186-187), and the 3^d neighbourhood sums sequentially in
// lexicographic offset order (grid.py:253-258).  Exact arithmetic differs
// from that by the reference's own rounding, and over long creeping runs
// (cfg4: 50 iterations) the trajectories drift apart by ~1e-9*h.  This
// header reproduces the reference's sums BIT FOR BIT, in parallel:
//
//  * A cell whose points all hold ONE value v (every cell after iteration 0
//    that received a single source cell: every point of a cell moves to the
//    same target, modeseek.py:109) sums c copies of v.  While the
//    accumulator stays in one binade [2^e, 2^(e+1)) every addition adds the
//    same number of ulps (round(v / ulp), ties to even: after the first tie
//    the accumulator is even and each tie adds round-up-to-even), so a whole
//    binade is one integer multiply-add; only the addition that crosses into
//    the next binade is done in fp64 -- O(log c) instead of O(c)
//    (seqsum_mag_from; pinned against np.add.accumulate by
//    tests/test_refsum_closed_form.py).
//  * A cell receiving several source cells ("mixed") needs its points in
//    index order: the points of mixed cells are stably radix-sorted by the
//    mixed cell's id (pass 0 streams the points in index order, so the sort
//    is stable in the index), then each cell is folded in order.  Long cells
//    are cut into 512-point windows: a window that provably stays inside one
//    binade is one integer add (its round(|v| / ulp) summed in parallel),
//    only windows holding a binade crossing are folded one point at a time.
//  * The first table (distinct input values) is exact whenever every value of
//    a cell is a multiple of the ulp of the cell's total (then no partial sum
//    rounds: checked per run); other runs take the same sort + fold.
// All values of one cell lie in [c*h, (c+1)*h) per axis, so they share one
// sign and the accumulator's magnitude grows monotonically: folds run on
// magnitudes and the sign is applied at the end (round-to-nearest-even is
// symmetric).
#pragma once

#include "gs_kernels.cuh"

namespace gs {

constexpr u32 kRsEmpty = 0xffffffffu;
constexpr u32 kRsPending = 0xfffffffeu;
constexpr u64 kMaxM = (1ull << 53) - 1;

// Device control block of the reference-order pipeline (one per context).
struct RsCtl {
  u32 nseg;       // segments to fold this round (mixed cells / inexact runs)
  u32 nelem;      // points of the segments that go through the global sort
  u32 npasses;    // radix passes over the segment ids (0: no global sort)
  u32 nbig;       // segments that go through the global sort
  u32 maxlen;     // longest segment (observability)
  u32 nsingle;    // single-source cells whose closed form was recomputed (not cached)
  u32 ncta;       // segments of kGatherWarp < len <= kGatherMax points (their ids: the CTA work list)
  u32 pad2;
};

// Index-ordered point lists of the cells (sorted runs only).  Every cell of
// table 0 is a run of the spatial sort, whose original indices perm[start,
// end) ascend (the sort is stable): that is its list.  A cell that moves as a
// whole keeps its list; a mixed target's list is the merge of its sources'
// lists, written to the arena behind perm -- so a mixed target is ordered by
// ranking each source's points among the other sources (binary searches),
// not by sorting all of its points again.  Lists: (offset << 32 | length)
// into `arena` (perm first), 0 = none (big segments, arena full): those
// cells' later merges fall back to the gather + sort of their runs.  The
// spatial sort places the points of a run in no particular order, so a run's
// own list is flagged raw (kListRaw in the length word) and is put in index
// order when a merge first loads it; published lists are ordered.
constexpr u32 kListRaw = 0x80000000u;

struct RsLists {
  bool on;            // source chains of the mixed targets (shead / snext)
  bool lists;         // cells carry point lists (cur / nxt / arena)
  const u64* cur;     // per slot of the source table
  u64* nxt;           // per slot of the target table
  u32* shead;         // per target slot: head of its source list (kRsEmpty-terminated)
  u32* snext;         // per source slot: next source of the same target
  u32* segdone;       // per segment: folded by a merge kernel
  u32* arena;         // perm, then published lists
  u64 cap;            // arena entries
  unsigned long long* top;   // next free arena entry
};

// Segments up to kGatherMax points (sorted runs) are gathered from their runs
// by one CTA and ordered in shared memory; longer ones (and every segment of
// an unsorted run) go through the global radix sort.
constexpr u32 kGatherMax = 8192;
constexpr u32 kGatherWarp = 256;   // gathered segments up to this size: one warp each

// ------------------------------------------------------- closed form

__host__ __device__ inline u64 dbits(double x) {
  u64 b;
  memcpy(&b, &x, sizeof b);
  return b;
}

__host__ __device__ inline double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}

// fl-sequential sum: starting from the magnitude s >= 0, add c copies of
// a >= 0, each addition rounded to nearest even -- exactly what c successive
// fp64 additions produce (s == 0 means the first addition is 0.0 + a).
__host__ __device__ inline double seqsum_mag_from(double s, double a, u64 c) {
  if (c == 0 || a == 0.0) return s;
  if (c == 1) return dadd(s, a);
  if (s == 0.0) {
    s = a;
    --c;
  }
  if (c <= 24) {                                    // a few copies: the additions themselves
    for (; c; --c) s = dadd(s, a);
    return s;
  }
  while (c) {
    const u64 sb = dbits(s);
    const int be = (int)(sb >> 52);                 // biased exponent (s > 0)
    if (be <= 1 || a < 0x1p-960) {                  // subnormal range: one by one
      for (; c; --c) s = dadd(s, a);
      break;
    }
    const int ue = be - 1075;                       // ulp(s) = 2^ue
    u64 m = (sb & ((1ull << 52) - 1)) | (1ull << 52);   // s = m * 2^ue
    const double x = scale2(a, -ue);                // a / ulp (exact scaling)
    if (x >= 0x1p52) {                              // a reaches s's binade: no fixed step
      s = dadd(s, a);
      --c;
      continue;
    }
    const double fl = floor(x);
    const double frac = x - fl;                     // exact
    const u64 q = (u64)fl;
    u64 delta;
    if (frac == 0.5) {
      // tie: the result is made even; afterwards m is even and every tie
      // adds q rounded up to even
      const u64 d1 = q + ((m + q) & 1ull);
      if (m + d1 > kMaxM) {
        s = dadd(s, a);
        --c;
        continue;
      }
      m += d1;
      --c;
      delta = q + (q & 1ull);
    } else {
      delta = frac > 0.5 ? q + 1 : q;
    }
    if (delta == 0) return scale2((double)m, ue);   // further additions change nothing
    // k = (kMaxM - m) / delta: both below 2^53, so the fp64 quotient is off by
    // at most one (cheaper than the 64-bit integer division)
    const u64 room = kMaxM - m;
    u64 k = (u64)((double)room / (double)delta);
    if (k * delta > room) --k;
    else if ((k + 1) * delta <= room) ++k;
    if (k > c) k = c;
    m += k * delta;
    c -= k;
    s = scale2((double)m, ue);
    if (c) {                                        // the crossing addition, in fp64
      s = dadd(s, a);
      --c;
    }
  }
  return s;
}

// np.bincount-order sum of c copies of v (from 0.0).
__host__ __device__ inline double seqsum_const(double v, u64 c) {
  const double r = seqsum_mag_from(0.0, fabs(v), c);
  return (v < 0.0 && r != 0.0) ? -r : r;
}

// ------------------------------------------------------- radix sort
// Stable LSD radix sort of (key, val) u32 pairs by 8-bit digits of the key.
// Pass 0 reads a virtual element stream (a functor over the index range
// [0, n0), invalid elements dropped -- the sort also compacts); later passes
// ping-pong between two buffers.  Tiles of 4096 elements per 256-thread
// block; warp w of a tile owns elements [512 w, 512 w + 512), item-major
// within the warp, so rank order == element order (stability).

constexpr int kRsThreads = 256, kRsItems = 8, kRsTile = kRsThreads * kRsItems;
constexpr int kRsWarps = kRsThreads / 32;

struct RsBufSrc {
  static constexpr bool kRunStream = false;
  const u32* keys;
  const u32* vals;
  const u32* n;       // element count (device)
  __device__ __forceinline__ i64 count() const { return (i64)*n; }
  __device__ __forceinline__ bool get(i64 i, u32& k, u32& v) const {
    k = keys[i];
    v = vals[i];
    return true;
  }
};

// Pass-0 stream: point i of run cell0[i] -> (key, value) of its run, one
// packed 8-byte gather (runkv: key low, value high; value ~0 = the point
// index i itself).
struct RsRunSrc {
  static constexpr bool kRunStream = true;
  const u32* cell0;
  const u64* runkv;
  i64 n;
  __device__ __forceinline__ i64 count() const { return n; }
  __device__ __forceinline__ bool get(i64 i, u32& k, u32& v) const {
    const u32 r = cell0[i];
    const u64 kv = r == kRsEmpty ? ~0ull : runkv[r];
    k = (u32)kv;
    v = (u32)(kv >> 32);
    if (v == kRsEmpty) v = (u32)i;
    return k != kRsEmpty;
  }
};

__device__ __forceinline__ bool rs_pass_live(const RsCtl* ctl, int pass) { return pass < (int)ctl->npasses; }

template <class Src>
__device__ __forceinline__ void rs_load_tile(const Src& src, i64 base, i64 n, u32 (&k)[kRsItems],
                                             u32 (&v)[kRsItems], bool (&ok)[kRsItems]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (Src::kRunStream) {
    // two phases so every item's run index is in flight before the gathers
    u32 r[kRsItems];
#pragma unroll
    for (int it = 0; it < kRsItems; ++it) {
      const i64 i = base + (i64)w * (32 * kRsItems) + it * 32 + lane;
      r[it] = i < n ? __ldcs(src.cell0 + i) : kRsEmpty;
    }
#pragma unroll
    for (int it = 0; it < kRsItems; ++it) {
      const i64 i = base + (i64)w * (32 * kRsItems) + it * 32 + lane;
      const u64 kv = r[it] == kRsEmpty ? ~0ull : src.runkv[r[it]];
      k[it] = (u32)kv;
      v[it] = (u32)(kv >> 32);
      if (v[it] == kRsEmpty) v[it] = (u32)i;
      ok[it] = k[it] != kRsEmpty;
    }
  } else {
#pragma unroll
    for (int it = 0; it < kRsItems; ++it) {
      const i64 i = base + (i64)w * (32 * kRsItems) + it * 32 + lane;
      ok[it] = false;
      k[it] = kRsEmpty;
      v[it] = 0;
      if (i < n) ok[it] = src.get(i, k[it], v[it]);
    }
  }
}

// per-tile digit counts, digit-major: counts[d * nblk + tile].  The grid is
// fixed (blocks loop over tiles), so a pass the device does not need costs one
// small launch.
template <class Src>
__global__ void __launch_bounds__(kRsThreads) k_rs_count(Src src, const RsCtl* ctl, int pass, u32* counts,
                                                         u32 nblk) {
  __shared__ u32 hist[256];
  if (!rs_pass_live(ctl, pass)) return;
  const i64 n = src.count();
  for (u32 tile = blockIdx.x; tile < nblk; tile += gridDim.x) {
    hist[threadIdx.x] = 0;
    __syncthreads();
    const i64 base = (i64)tile * kRsTile;
    if (base < n) {
      u32 k[kRsItems], v[kRsItems];
      bool ok[kRsItems];
      rs_load_tile(src, base, n, k, v, ok);
#pragma unroll
      for (int it = 0; it < kRsItems; ++it) {
        const u32 d = ok[it] ? (k[it] >> (8 * pass)) & 255u : 256u;
        const unsigned peers = __match_any_sync(kFull, d);
        if (d < 256u && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[d], (u32)__popc(peers));
      }
    }
    __syncthreads();
    counts[(size_t)threadIdx.x * nblk + tile] = hist[threadIdx.x];
  }
}

// exclusive scan of a u32 array (three kernels: chunk sums, top, apply)
constexpr int kScan32Chunk = 4096;
__global__ void __launch_bounds__(256) k_scan32_reduce(const u32* a, i64 n, u32* sums, const RsCtl* ctl, int pass) {
  if (ctl && !rs_pass_live(ctl, pass)) return;
  const i64 b0 = (i64)blockIdx.x * kScan32Chunk;
  u32 s = 0;
  for (i64 i = b0 + threadIdx.x; i < min(n, b0 + kScan32Chunk); i += 256) s += a[i];
  s = __reduce_add_sync(kFull, s);
  __shared__ u32 ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 t = 0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan32_top(u32* sums, int nb, const RsCtl* ctl, int pass) {
  if (ctl && !rs_pass_live(ctl, pass)) return;
  __shared__ u32 ws[32];
  __shared__ u32 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const u32 x = i < nb ? sums[i] : 0u;
    u32 incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(kFull, incl, o);
      if ((threadIdx.x & 31) >= o) incl += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = incl;
    __syncthreads();
    if (threadIdx.x < 32) {
      u32 w = ws[threadIdx.x], wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(kFull, wi, o);
        if (threadIdx.x >= o) wi += y;
      }
      ws[threadIdx.x] = wi - w;
    }
    __syncthreads();
    const u32 excl = carry + ws[threadIdx.x >> 5] + incl - x;
    __syncthreads();
    if (i < nb) sums[i] = excl;
    if (threadIdx.x == 1023) carry = excl + x;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_scan32_apply(u32* a, i64 n, const u32* sums, const RsCtl* ctl, int pass) {
  if (ctl && !rs_pass_live(ctl, pass)) return;
  const i64 b0 = (i64)blockIdx.x * kScan32Chunk;
  const i64 b1 = min(n, b0 + kScan32Chunk);
  __shared__ u32 ws[8];
  __shared__ u32 carry;
  if (threadIdx.x == 0) carry = sums[blockIdx.x];
  __syncthreads();
  for (i64 c0 = b0; c0 < b1; c0 += 256) {
    const i64 i = c0 + threadIdx.x;
    const u32 x = i < b1 ? a[i] : 0u;
    u32 incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(kFull, incl, o);
      if ((threadIdx.x & 31) >= o) incl += y;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = incl;
    __syncthreads();
    u32 wb = 0;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) wb += ws[w];
    if (i < b1) a[i] = carry + wb + incl - x;
    __syncthreads();
    if (threadIdx.x == 255) carry += wb + incl;
    __syncthreads();
  }
}

// stable scatter by digit: offsets = scanned counts.  The tile is first
// ordered by digit in shared memory (stable), then written out with
// consecutive threads on consecutive positions of each digit's run, so the
// global writes coalesce instead of scattering 4-byte stores.
template <class Src>
__global__ void __launch_bounds__(kRsThreads, 4) k_rs_scatter(Src src, const RsCtl* ctl, int pass, const u32* offs,
                                                              u32 nblk, u32* okeys, u32* ovals) {
  __shared__ u32 base[kRsWarps][256];
  __shared__ u32 tdig[257];      // the tile's exclusive digit offsets
  __shared__ u32 gofs[256];      // global offset of (digit, tile)
  __shared__ u32 sk[kRsTile];
  __shared__ u32 sv[kRsTile];
  __shared__ u32 ws[kRsWarps];
  if (!rs_pass_live(ctl, pass)) return;
  const i64 n = src.count();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (u32 tile = blockIdx.x; tile < nblk; tile += gridDim.x) {
  const i64 t0 = (i64)tile * kRsTile;
  if (t0 >= n) break;
  __syncthreads();   // the previous tile's shared arrays are done with
  for (int q = threadIdx.x; q < kRsWarps * 256; q += kRsThreads) (&base[0][0])[q] = 0;
  __syncthreads();
  u32 k[kRsItems], v[kRsItems];
  bool ok[kRsItems];
  rs_load_tile(src, t0, n, k, v, ok);
  u32 dg[kRsItems];
#pragma unroll
  for (int it = 0; it < kRsItems; ++it) {
    dg[it] = ok[it] ? (k[it] >> (8 * pass)) & 255u : 256u;
    const unsigned peers = __match_any_sync(kFull, dg[it]);
    if (dg[it] < 256u && lane == __ffs(peers) - 1) base[w][dg[it]] += (u32)__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  u32 tot;
  {
    // digit d: warp bases inside the tile's digit run; the tile's count
    const int d = threadIdx.x;
    u32 acc = 0;
#pragma unroll
    for (int ww = 0; ww < kRsWarps; ++ww) {
      const u32 c = base[ww][d];
      base[ww][d] = acc;
      acc += c;
    }
    tot = acc;
    gofs[d] = offs[(size_t)d * nblk + tile];
  }
  // exclusive scan of the tile's digit counts (256 threads = 256 digits)
  {
    u32 inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    u32 wb = 0;
    for (int ww = 0; ww < w; ++ww) wb += ws[ww];
    tdig[threadIdx.x] = wb + inc - tot;
    if (threadIdx.x == 255) tdig[256] = wb + inc;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < kRsItems; ++it) {
    const unsigned peers = __match_any_sync(kFull, dg[it]);
    u32 pos = 0;
    if (dg[it] < 256u) pos = tdig[dg[it]] + base[w][dg[it]] + (u32)__popc(peers & lt);
    __syncwarp();
    if (dg[it] < 256u && lane == __ffs(peers) - 1) base[w][dg[it]] += (u32)__popc(peers);
    __syncwarp();
    if (dg[it] < 256u) {
      sk[pos] = k[it];
      sv[pos] = v[it];
    }
  }
  __syncthreads();
  const u32 nt = tdig[256];
  for (u32 e = threadIdx.x; e < nt; e += kRsThreads) {
    const u32 kk = sk[e];
    const u32 d = (kk >> (8 * pass)) & 255u;
    const u32 out = gofs[d] + (e - tdig[d]);
    okeys[out] = kk;
    ovals[out] = sv[e];
  }
  }
}

// The sorted pairs: pass p writes buffer p & 1, so the result sits in
// buffer (npasses - 1) & 1 (npasses is known on device only).
struct RsSorted {
  const u32* k0;
  const u32* v0;
  const u32* k1;
  const u32* v1;
  __device__ __forceinline__ const u32* keys(const RsCtl* c) const { return ((c->npasses - 1) & 1) ? k1 : k0; }
  __device__ __forceinline__ const u32* vals(const RsCtl* c) const { return ((c->npasses - 1) & 1) ? v1 : v0; }
};

// segment bounds of the sorted keys: start[key], end[key]
__global__ void __launch_bounds__(256) k_rs_bounds(RsSorted so, const RsCtl* ctl, u32* sstart, u32* send) {
  if (ctl->npasses == 0) return;
  const u32* keys = so.keys(ctl);
  const i64 n = ctl->nelem;
  for (i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (i64)gridDim.x * blockDim.x) {
    const u32 k = keys[p];
    if (p == 0 || keys[p - 1] != k) sstart[k] = (u32)p;
    if (p == n - 1 || keys[p + 1] != k) send[k] = (u32)(p + 1);
  }
}

// number of 8-bit passes for keys < nseg
__global__ void k_rs_passes(RsCtl* ctl) {
  const u32 ns = ctl->nseg;
  u32 p = 0;
  if (ns > 0 && ctl->nbig > 0) {
    const u32 mx = ns - 1;
    p = mx < 256u ? 1 : mx < 65536u ? 2 : mx < (1u << 24) ? 3 : 4;
  }
  ctl->npasses = p;
}

// ------------------------------------------------------- ordered folds
// A fold target: segment id q -> output slot, value source for its sorted
// elements, per-axis sign (all values of a cell share it).

constexpr int kFoldWin = 512;          // window of the parallel path
constexpr u32 kFoldBig = 4 * kFoldWin;  // segments longer than this use windows
constexpr u64 kNoDelta = ~0ull;

// value of sorted element p on axis j: iteration folds read the source
// cell's target record (rec[val].t[j]); first-table folds the input value
// of point val (original order)
template <int D>
struct RecVal {
  const Rec<D>* rec;
  __device__ __forceinline__ double get(u32 val, int j) const { return rec[val].t[j]; }
};

template <int D>
struct InVal {
  const void* p;
  int kind;    // 0: fp64 AoS (n, D), 1: fp32 AoS, 2: fp64 SoA (ld)
  i64 ld;
  __device__ __forceinline__ double get(u32 i, int j) const {
    if (kind == 0) return static_cast<const double*>(p)[(i64)i * D + j];
    if (kind == 1) return (double)static_cast<const float*>(p)[(i64)i * D + j];
    return static_cast<const double*>(p)[(i64)j * ld + i];
  }
};

// window pass 1: per full window inside one long segment, the approximate
// per-axis magnitude sum (any order); others marked invalid
template <int D, class Val>
__global__ void __launch_bounds__(256) k_fold_win(RsSorted so, const RsCtl* ctl, const u32* sstart, const u32* send,
                                                  Val V, double* wsum) {
  if (ctl->npasses == 0) return;
  const u32* __restrict__ keys = so.keys(ctl);
  const u32* __restrict__ vals = so.vals(ctl);
  const i64 n = ctl->nelem;
  const i64 nw = n / kFoldWin;
  const int lane = threadIdx.x & 31;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 w = warp; w < nw; w += nwarps) {
    const i64 p0 = w * kFoldWin;
    const u32 k0 = keys[p0];
    bool full = keys[p0 + kFoldWin - 1] == k0 && send[k0] - sstart[k0] > kFoldBig;
    double s[D];
#pragma unroll
    for (int j = 0; j < D; ++j) s[j] = 0.0;
    if (full) {
      for (int q = lane; q < kFoldWin; q += 32) {
        const u32 v = vals[p0 + q];
#pragma unroll
        for (int j = 0; j < D; ++j) s[j] += fabs(V.get(v, j));
      }
#pragma unroll
      for (int j = 0; j < D; ++j)
        for (int o = 16; o; o >>= 1) s[j] += __shfl_xor_sync(kFull, s[j], o);
    }
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < D; ++j) wsum[w * D + j] = full ? s[j] : -1.0;
  }
}

// window pass 2: per long segment (one warp), the approximate accumulator
// before each of its full windows (prefix of the window sums)
template <int D, class Val>
__global__ void __launch_bounds__(256) k_fold_pre(RsSorted so, const RsCtl* ctl, const u32* sstart,
                                                  const u32* send, Val V, const double* wsum, double* wpre) {
  if (ctl->npasses == 0) return;
  const u32* __restrict__ vals = so.vals(ctl);
  const u32 nseg = ctl->nseg;
  const int lane = threadIdx.x & 31;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 q = warp; q < nseg; q += nwarps) {
    const u32 a = sstart[q], b = send[q];
    if (b - a <= kFoldBig) continue;
    const u32 w0 = (a + kFoldWin - 1) / kFoldWin, w1 = b / kFoldWin;   // full windows [w0, w1)
    double acc[D];
#pragma unroll
    for (int j = 0; j < D; ++j) acc[j] = 0.0;
    for (u32 p = a + lane; p < w0 * kFoldWin; p += 32) {
      const u32 v = vals[p];
#pragma unroll
      for (int j = 0; j < D; ++j) acc[j] += fabs(V.get(v, j));
    }
#pragma unroll
    for (int j = 0; j < D; ++j)
      for (int o = 16; o; o >>= 1) acc[j] += __shfl_xor_sync(kFull, acc[j], o);
    for (u32 w = w0; w < w1; w += 32) {
      const u32 ww = w + lane;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double x = ww < w1 ? wsum[(i64)ww * D + j] : 0.0;
        double incl = x;
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += y;
        }
        if (ww < w1) wpre[(i64)ww * D + j] = acc[j] + incl - x;
        acc[j] += __shfl_sync(kFull, incl, 31);
      }
    }
  }
}

// window pass 3: a window whose accumulator range provably stays in one
// binade adds sum_i round(|v_i| / ulp) ulps -- precomputed here in
// parallel; windows holding a crossing or a tie stay kNoDelta
template <int D, class Val>
__global__ void __launch_bounds__(256) k_fold_delta(RsSorted so, const RsCtl* ctl, Val V,
                                                    const double* wsum, const double* wpre, u64* wdelta) {
  if (ctl->npasses == 0) return;
  const u32* __restrict__ vals = so.vals(ctl);
  const i64 nw = (i64)ctl->nelem / kFoldWin;
  const int lane = threadIdx.x & 31;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 w = warp; w < nw; w += nwarps) {
    // per axis: the binade the window's accumulator provably stays in
    // (|accumulator - prefix| <= elements so far * 2^-53 * accumulator;
    // 2^-20 covers any segment below 2^32 points)
    int ue[D];
    bool live[D], any = false;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double ws = wsum[w * D + j];
      live[j] = false;
      ue[j] = 0;
      if (ws >= 0.0) {
        const double lo = wpre[w * D + j] * (1.0 - 0x1p-20);
        const double hi = (wpre[w * D + j] + ws) * (1.0 + 0x1p-20);
        const int blo = (int)(dbits(lo) >> 52), bhi = (int)(dbits(hi) >> 52);
        if (lo > 0x1p-900 && blo == bhi && bhi < 2047) {
          live[j] = true;
          ue[j] = blo - 1075;
          any = true;
        }
      }
    }
    u64 sum[D];
    bool tie[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { sum[j] = 0; tie[j] = false; }
    if (any) {
      for (int q = lane; q < kFoldWin; q += 32) {
        const u32 vv = vals[w * kFoldWin + q];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if (!live[j]) continue;
          const double x = scale2(fabs(V.get(vv, j)), -ue[j]);
          const double fl = floor(x);
          const double fr = x - fl;
          tie[j] |= fr == 0.5;
          sum[j] += (u64)fl + (fr > 0.5 ? 1ull : 0ull);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      for (int o = 16; o; o >>= 1) sum[j] += __shfl_xor_sync(kFull, sum[j], o);
      const bool t = __any_sync(kFull, tie[j]);
      // tag: the biased exponent of the binade the step is valid in (11
      // bits above the 53-bit step)
      const u64 res = (live[j] && !t && sum[j] <= kMaxM) ? (((u64)(ue[j] + 1075) << 53) | sum[j]) : kNoDelta;
      if (lane == 0) wdelta[w * D + j] = res;
    }
  }
}

// Warp-cooperative fold of elements [a, b) into the magnitude s (uniform
// across the warp): 32 elements at a time, each converted to its integer
// step round(|v| / ulp) in the accumulator's current binade; a warp scan of
// the steps commits every element before the first one that would leave the
// binade (or is a tie), that one is added in fp64, and the next chunk
// starts right after it.  Exactly the sequential fp64 sum, at ~1 warp scan
// per 32 elements instead of 32 dependent additions.
template <int D, class Val, class VT = u32>
__device__ __forceinline__ double warp_fold(double s, const VT* __restrict__ vals, u32 a, u32 b, const Val& V, int j) {
  const int lane = threadIdx.x & 31;
  u32 i = a;
  u32 have = 0xffffffffu;   // chunk start the prefetched values belong to
  double nxt = 0.0;
  while (i < b) {
    const u32 idx = i + lane;
    const bool valid = idx < b;
    const double av = (have == i) ? nxt : (valid ? fabs(V.get(vals[idx], j)) : 0.0);
    // the next chunk's values, in flight while this one is reduced
    have = i + 32;
    nxt = (i + 32 + lane < b) ? fabs(V.get(vals[i + 32 + lane], j)) : 0.0;
    if (s == 0.0) {            // first addition of the segment: 0.0 + v is exact
      s = __shfl_sync(kFull, av, 0);
      i += 1;
      continue;
    }
    const u64 sb = dbits(s);
    const int be = (int)(sb >> 52);
    if (be <= 1) {             // subnormal accumulator (never in practice): one at a time
      s = __dadd_rn(s, __shfl_sync(kFull, av, 0));
      i += 1;
      continue;
    }
    const int ue = be - 1075;
    const u64 m = (sb & ((1ull << 52) - 1)) | (1ull << 52);
    bool bad = false;
    u64 dl = 0;
    if (valid) {
      const double x = scale2(av, -ue);
      if (x >= 0x1p52) {
        bad = true;
      } else {
        const double fl = floor(x);
        const double fr = x - fl;
        bad = fr == 0.5;
        dl = (u64)fl + (fr > 0.5 ? 1ull : 0ull);
      }
    }
    u64 inc = dl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u64 y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    const unsigned stop = __ballot_sync(kFull, valid && (bad || m + inc > kMaxM));
    if (stop == 0) {
      s = scale2((double)(m + __shfl_sync(kFull, inc, 31)), ue);
      i += 32;
      continue;
    }
    const int L = __ffs(stop) - 1;
    const u64 before = __shfl_sync(kFull, inc, L > 0 ? L - 1 : 0);
    s = scale2((double)(m + (L > 0 ? before : 0ull)), ue);
    s = __dadd_rn(s, __shfl_sync(kFull, av, L));
    i += (u32)L + 1;
  }
  return s;
}

constexpr u32 kFoldSmall = 256;   // segments up to this length: one thread per (segment, axis)

// the fold, short segments: one thread per (segment, axis), plain
// sequential additions, loads batched ahead of the dependent adds
template <int D, class Val>
__global__ void __launch_bounds__(256) k_fold_small(RsSorted so, const RsCtl* ctl, const u32* sstart,
                                                    const u32* send, Val V, const u32* outslot, double* rs) {
  if (ctl->npasses == 0) return;
  const u32* __restrict__ vals = so.vals(ctl);
  const i64 items = (i64)ctl->nseg * D;
  for (i64 it = (i64)blockIdx.x * blockDim.x + threadIdx.x; it < items; it += (i64)gridDim.x * blockDim.x) {
    const u32 q = (u32)(it / D);
    const int j = (int)(it % D);
    const u32 a = sstart[q], b = send[q];
    if (b == a || b - a > kFoldSmall) continue;   // gathered segment / long one
    double s = 0.0;
    bool neg = false;
    for (u32 i = a; i < b; i += 8) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = (i + k < b) ? V.get(vals[i + k], j) : 0.0;
      if (i == a) neg = v[0] < 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i + k < b) s = __dadd_rn(s, fabs(v[k]));
    }
    rs[(i64)outslot[q] * D + j] = (neg && s != 0.0) ? -s : s;
  }
}

// the fold, long segments: one warp per (segment, axis); the precomputed
// window steps where the accumulator really is in the binade the step was
// computed for, warp_fold everywhere else
template <int D, class Val>
__global__ void __launch_bounds__(256) k_fold_big(RsSorted so, const RsCtl* ctl, const u32* sstart,
                                                  const u32* send, Val V, const u64* wdelta, const u32* outslot,
                                                  double* rs) {
  if (ctl->npasses == 0) return;
  const u32* __restrict__ vals = so.vals(ctl);
  const i64 items = (i64)ctl->nseg * D;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 it = warp; it < items; it += nwarps) {
    const u32 q = (u32)(it / D);
    const int j = (int)(it % D);
    const u32 a = sstart[q], b = send[q];
    if (b - a <= kFoldSmall) continue;
    const bool neg = V.get(vals[a], j) < 0.0;
    double s = 0.0;
    if (b - a <= kFoldBig) {
      s = warp_fold<D>(s, vals, a, b, V, j);
    } else {
      const u32 w0 = (a + kFoldWin - 1) / kFoldWin, w1 = b / kFoldWin;
      s = warp_fold<D>(s, vals, a, w0 * kFoldWin, V, j);
      const int lane = threadIdx.x & 31;
      for (u32 wb = w0; wb < w1; wb += 32) {
        // 32 window steps at once (lane l holds window wb + l)
        const u64 mine = (wb + lane < w1) ? wdelta[(i64)(wb + lane) * D + j] : kNoDelta;
        const u32 wn = min(32u, w1 - wb);
        for (u32 k = 0; k < wn; ++k) {
          const u64 dt = __shfl_sync(kFull, mine, k);
          const u64 sb = dbits(s);
          if (dt != kNoDelta && s > 0.0 && (u64)(sb >> 52) == (dt >> 53)) {
            const u64 m = (sb & ((1ull << 52) - 1)) | (1ull << 52);
            const u64 dm = dt & kMaxM;
            if (m + dm <= kMaxM) {
              s = scale2((double)(m + dm), (int)(sb >> 52) - 1075);
              continue;
            }
          }
          const u32 w = wb + k;
          s = warp_fold<D>(s, vals, w * kFoldWin, (w + 1) * kFoldWin, V, j);
        }
      }
      s = warp_fold<D>(s, vals, w1 * kFoldWin, b, V, j);
    }
    if ((threadIdx.x & 31) == 0) rs[(i64)outslot[q] * D + j] = (neg && s != 0.0) ? -s : s;
  }
}

// ------------------------------------------------------- table chain hooks

// Sources of table t: every occupied cell s with its target record.  A
// target reached by exactly one source holds count_s copies of that
// source's target value: closed form.  Other targets become fold segments
// (ids in first-come order; the ids only key the sort).
template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_rs_classify(GridParams g, Tab cur, Tab nxt, const Rec<D>* __restrict__ rec,
                                                          Ctrl* ctrl, int c, int t, const u32* nsrc, u32* mid,
                                                          u32* outslot, double* rs_next, RsCtl* rsc, u32* seglen,
                                                          u32* sstart, u32* send, bool all_big, Rec<D>* tag,
                                                          RsLists L, u32* ctalist) {
  if (block_stopped_before(ctrl, t)) return;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const i64 items = Tab::kDense ? (i64)g.nkeys : (i64)ctrl->k[c];
  u32 nrecomp = 0;
  for (i64 a = tid; a < items; a += stride) {
    const u32 s = Tab::kDense ? (u32)a : cur.list[a];
    const u64 cnt = cur.ent[s].count;
    if (cnt == 0) continue;
    const Rec<D> r = rec[s];
    const u32 ts = nxt.lookup(r.key);
    if (nsrc[ts] == 1) {
      // the buffer already holds seqsum(t, cnt) for this slot when its tag
      // (the value and count it was computed from) matches: converged cells
      // repeat theirs every other iteration
      Rec<D> tg = tag[ts];
      bool same = tg.key == cnt;
#pragma unroll
      for (int j = 0; j < D; ++j) same &= dbits(tg.t[j]) == dbits(r.t[j]);
      if (!same) {
#pragma unroll
        for (int j = 0; j < D; ++j) rs_next[(i64)ts * D + j] = seqsum_const(r.t[j], cnt);
        tg = r;
        tg.key = cnt;
        tag[ts] = tg;
        ++nrecomp;
      }
      if (L.lists) L.nxt[ts] = L.cur[s];   // the cell's index-ordered point list moves with it
    } else {
      if (L.on) L.snext[s] = atomicExch(L.shead + ts, s);   // source list of the mixed target
      if (atomicCAS(mid + ts, kRsEmpty, kRsPending) != kRsEmpty) continue;
      const u32 m = atomicAdd(&rsc->nseg, 1u);
      const u32 len = (u32)nxt.ent[ts].count;
      outslot[m] = ts;
      seglen[m] = len;
      sstart[m] = 0;
      send[m] = 0;
      if (L.lists) {
        L.nxt[ts] = 0;       // no list unless a merge publishes one
        L.segdone[m] = 0;
      }
      tag[ts].key = 0;   // the fold writes this slot: no cached closed form
      atomicMax(&rsc->maxlen, len);
      if (all_big || len > kGatherMax) {
        atomicAdd(&rsc->nelem, len);
        atomicAdd(&rsc->nbig, 1u);
      } else if (ctalist && len > kGatherWarp) {
        ctalist[atomicAdd(&rsc->ncta, 1u)] = m;
      }
      mid[ts] = m;
    }
  }
  nrecomp = __reduce_add_sync(kFull, nrecomp);
  if ((threadIdx.x & 31) == 0 && nrecomp) atomicAdd(&rsc->nsingle, nrecomp);
}

// Per run (initial cell): its current cell moves to the target's slot; the
// run's points are fold elements (key = segment id) when that slot is mixed,
// with the source slot as value.
template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_rs_runs(const u32* runs, const u32* nruns, const u32* rc_cur, u32* rc_nxt,
                                                      const Rec<D>* __restrict__ rec, Tab nxt, const u32* mid,
                                                      u32* runkey, u32* runval, Ctrl* ctrl, int t, const u32* seglen,
                                                      u32* runseg, u32* segbeg, bool all_big, u64* runkv) {
  if (block_stopped_before(ctrl, t)) return;
  const u32 nr = *nruns;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < nr; a += (i64)gridDim.x * blockDim.x) {
    const u32 r = runs[a];
    const u32 src = rc_cur[r];
    const u32 ts = nxt.lookup(rec[src].key);
    rc_nxt[r] = ts;
    const u32 q = mid[ts];
    const bool big = q != kRsEmpty && (all_big || seglen[q] > kGatherMax);
    runkey[r] = big ? q : kRsEmpty;      // global sort: points of long segments
    runval[r] = src;
    runkv[r] = ((u64)src << 32) | (big ? q : kRsEmpty);
    runseg[a] = (q != kRsEmpty && !big) ? q : kRsEmpty;   // gathered segments: their runs
    if (q != kRsEmpty && !big) atomicAdd(segbeg + q, 1u);   // counts; scanned into offsets
  }
}

// run lists of the gathered segments: seglist[segbeg[q] ...] (segbeg = the
// exclusive scan of segcnt; segcur zero on entry)
__global__ void __launch_bounds__(kThreads) k_rs_fill(const u32* runs, const u32* nruns, const u32* runseg,
                                                      const u32* segbeg, u32* segcur, u32* seglist) {
  const u32 nr = *nruns;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < nr; a += (i64)gridDim.x * blockDim.x) {
    const u32 q = runseg[a];
    if (q == kRsEmpty) continue;
    seglist[segbeg[q] + atomicAdd(segcur + q, 1u)] = runs[a];
  }
}

constexpr size_t kGatherWarpSmem = (size_t)8 * 2 * kGatherWarp * sizeof(u32);

// One warp per gathered segment of <= kGatherWarp points (the common case
// once clusters contract): run offsets by a warp scan, points' original
// indices and values into the warp's shared-memory slice, warp-synchronous
// bitonic sort by index, then warp_fold per axis.
template <int D, class Val, bool kFirst>
__global__ void __launch_bounds__(256) k_rs_gather_warp(const RsCtl* ctl, const u32* seglen, const u32* segbeg,
                                                        const u32* seglist, const u32* start, const u32* end,
                                                        const u32* perm, const u32* runval, Val V,
                                                        const u32* outslot, double* rs, bool all_big, RsLists L) {
  extern __shared__ u32 wsm[];
  if (all_big) return;
  const u32 nseg = ctl->nseg;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u32* xi = wsm + (size_t)w * 2 * kGatherWarp;
  u32* xv = xi + kGatherWarp;
  const i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 q = gw; q < nseg; q += nw) {
    const u32 len = seglen[q];
    if (len == 0 || len > kGatherWarp) continue;   // warp-uniform
    if (!kFirst && L.lists && L.segdone[q]) continue;   // folded by a list merge
    const u32 b0 = segbeg ? segbeg[q] : (u32)q;
    const u32 nr = segbeg ? segbeg[q + 1] - b0 : 1u;
    // runs: lane k copies run k, k+32, ... at its exclusive offset
    u32 carry = 0;
    for (u32 k0 = 0; k0 < nr; k0 += 32) {
      const u32 k = k0 + lane;
      u32 r = 0, p0 = 0, l = 0;
      if (k < nr) {
        r = seglist[b0 + k];
        p0 = start[r];
        l = end[r] - p0;
      }
      u32 inc = l;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
      }
      const u32 off = carry + inc - l;
      const u32 rv = (kFirst || k >= nr) ? 0u : runval[r];
      for (u32 e = 0; e < l; ++e) {
        const u32 idx = perm[p0 + e];
        xi[off + e] = idx;
        xv[off + e] = kFirst ? idx : rv;
      }
      carry += __shfl_sync(kFull, inc, 31);
    }
    u32 P = 1;
    while (P < len) P <<= 1;
    for (u32 e = len + lane; e < P; e += 32) {
      xi[e] = 0xffffffffu;
      xv[e] = 0;
    }
    __syncwarp();
    for (u32 k = 2; k <= P; k <<= 1)
      for (u32 jj = k >> 1; jj > 0; jj >>= 1) {
        for (u32 e = lane; e < P; e += 32) {
          const u32 x = e ^ jj;
          if (x > e) {
            const u32 a = xi[e], b = xi[x];
            if ((a > b) == ((e & k) == 0)) {
              xi[e] = b;
              xi[x] = a;
              const u32 va = xv[e];
              xv[e] = xv[x];
              xv[x] = va;
            }
          }
        }
        __syncwarp();
      }
    if (!kFirst && L.lists) {   // the sorted indices are the target's list
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(L.top, (unsigned long long)len);
      at = __shfl_sync(kFull, at, 0);
      if (at + len <= L.cap) {
        for (u32 e = lane; e < len; e += 32) L.arena[at + e] = xi[e];
        if (lane == 0) L.nxt[outslot[q]] = (at << 32) | len;
      }
    }
#pragma unroll 1
    for (int j = 0; j < D; ++j) {
      const bool neg = V.get(xv[0], j) < 0.0;
      const double sm = warp_fold<D>(0.0, xv, 0, len, V, j);
      if (lane == 0) rs[(i64)outslot[q] * D + j] = (neg && sm != 0.0) ? -sm : sm;
    }
    __syncwarp();
  }
}

// One CTA per gathered segment (<= kGatherMax points, made of whole runs of
// the spatial sort): its points' original indices (perm) and values are
// collected in shared memory, bitonic-sorted by index (= np.bincount's
// order), then warp j < D folds axis j with warp_fold.
constexpr size_t kGatherSmem = (size_t)(3 * kGatherMax + 1) * sizeof(u32);

template <int D, class Val, bool kFirst>
__global__ void __launch_bounds__(256) k_rs_gather(const RsCtl* ctl, const u32* seglen, const u32* segbeg,
                                                   const u32* seglist, const u32* start,
                                                   const u32* end, const u32* perm, const u32* runval, Val V,
                                                   const u32* outslot, double* rs, bool all_big, RsLists L,
                                                   const u32* ctalist) {
  extern __shared__ u32 gsm[];
  u32* sidx = gsm;
  u32* sval = gsm + kGatherMax;
  u32* roff = gsm + 2 * kGatherMax;
  __shared__ u32 wsum[8];
  __shared__ unsigned long long pub_at;
  if (all_big) return;
  const u32 nwork = ctalist ? ctl->ncta : ctl->nseg;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (u32 wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
    const u32 q = ctalist ? ctalist[wi] : wi;
    const u32 len = seglen[q];
    if (len <= kGatherWarp || len > kGatherMax) continue;   // block-uniform
    if (!kFirst && L.lists && L.segdone[q]) continue;          // folded by a list merge
    const u32 b0 = segbeg ? segbeg[q] : q;
    const u32 nr = segbeg ? segbeg[q + 1] - b0 : 1u;
    // exclusive offsets of the segment's runs (block scan of their lengths)
    u32 carry = 0;
    for (u32 k0 = 0; k0 < nr; k0 += 256) {
      const u32 k = k0 + tid;
      u32 l = 0;
      if (k < nr) {
        const u32 r = seglist[b0 + k];
        l = end[r] - start[r];
      }
      u32 inc = l;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) wsum[w] = inc;
      __syncthreads();
      u32 wb = 0, tot = 0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) {
        wb += ww < w ? wsum[ww] : 0u;
        tot += wsum[ww];
      }
      if (k < nr) roff[k] = carry + wb + inc - l;
      carry += tot;
      __syncthreads();
    }
    // gather: a warp per run
    for (u32 k = w; k < nr; k += 8) {
      const u32 r = seglist[b0 + k];
      const u32 p0 = start[r], p1 = end[r], o = roff[k];
      const u32 rv = kFirst ? 0u : runval[r];
      for (u32 pp = p0 + lane; pp < p1; pp += 32) {
        const u32 idx = perm[pp];
        sidx[o + pp - p0] = idx;
        sval[o + pp - p0] = kFirst ? idx : rv;
      }
    }
    u32 P = 1;
    while (P < len) P <<= 1;
    for (u32 e = len + tid; e < P; e += 256) {
      sidx[e] = 0xffffffffu;
      sval[e] = 0;
    }
    __syncthreads();
    // bitonic sort by original index
    for (u32 k = 2; k <= P; k <<= 1)
      for (u32 jj = k >> 1; jj > 0; jj >>= 1) {
        for (u32 e = tid; e < P; e += 256) {
          const u32 x = e ^ jj;
          if (x > e) {
            const u32 a = sidx[e], b = sidx[x];
            if ((a > b) == ((e & k) == 0)) {
              sidx[e] = b;
              sidx[x] = a;
              const u32 va = sval[e];
              sval[e] = sval[x];
              sval[x] = va;
            }
          }
        }
        __syncthreads();
      }
    if (!kFirst && L.lists) {   // the sorted indices are the target's list
      if (tid == 0) pub_at = atomicAdd(L.top, (unsigned long long)len);
      __syncthreads();
      const unsigned long long at = pub_at;
      if (at + len <= L.cap) {
        for (u32 e = tid; e < len; e += 256) L.arena[at + e] = sidx[e];
        if (tid == 0) L.nxt[outslot[q]] = (at << 32) | len;
      }
    }
    if (w < D) {
      const bool neg = V.get(sval[0], w) < 0.0;
      const double sm = warp_fold<D>(0.0, sval, 0, len, V, w);
      if (lane == 0) rs[(i64)outslot[q] * D + w] = (neg && sm != 0.0) ? -sm : sm;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- list merges

// values of a merge: the sources' target coordinates, staged in shared memory
struct LocVal {
  const double* t;   // [source][D]
  int d;
  __device__ __forceinline__ double get(u32 k, int j) const { return t[k * d + j]; }
};

// number of entries of the ascending list a[0, n) below x
__device__ __forceinline__ u32 list_rank(const u32* a, u32 n, u32 x) {
  if (n == 0 || x < a[0]) return 0;
  if (x > a[n - 1]) return n;
  u32 lo = 0, hi = n;
  while (lo < hi) {
    const u32 m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1; else hi = m;
  }
  return lo;
}

constexpr u32 kMergeWarpSrc = 32;    // sources a warp merge handles
constexpr size_t merge_warp_smem(int d) {
  // per warp: in (256 u32), out (256 u32), source number (256 u8), offsets (33 u32), values (32 x d f64)
  return (size_t)8 * (2 * kGatherWarp * 4 + kGatherWarp + 36 * 4 + kMergeWarpSrc * d * 8);
}

// One warp per mixed segment of <= kGatherWarp points whose sources all carry
// lists: rank-merge, publish the merged list, fold in index order.
template <int D>
__global__ void __launch_bounds__(256) k_rs_merge_warp(const RsCtl* ctl, const u32* seglen, const u32* outslot,
                                                       const Rec<D>* __restrict__ rec, RsLists L, double* rs) {
  extern __shared__ __align__(16) unsigned char msm[];
  const u32 nseg = ctl->nseg;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr size_t per = 2 * kGatherWarp * 4 + kGatherWarp + 36 * 4 + kMergeWarpSrc * D * 8;
  unsigned char* base = msm + (size_t)w * per;
  double* tv = reinterpret_cast<double*>(base);                       // 32 x D
  u32* xin = reinterpret_cast<u32*>(base + kMergeWarpSrc * D * 8);     // 256
  u32* xout = xin + kGatherWarp;                                       // 256
  u32* soff = xout + kGatherWarp;                                      // 33 (+3 pad)
  unsigned char* xk = reinterpret_cast<unsigned char*>(soff + 36);     // 256
  const i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 q = gw; q < nseg; q += nw) {
    const u32 len = seglen[q];
    if (len == 0 || len > kGatherWarp) continue;   // warp-uniform
    const u32 ts = outslot[q];
    // the sources: lane k takes the k-th of the chain
    u32 mysrc = kRsEmpty, m = 0;
    {
      u32 s = L.shead[ts];
      while (s != kRsEmpty && m < kMergeWarpSrc) {
        if ((u32)lane == m) mysrc = s;
        s = L.snext[s];
        ++m;
      }
      if (s != kRsEmpty) continue;                 // more sources than lanes: the gather path
    }
    const u64 lst = (u32)lane < m ? L.cur[mysrc] : 0ull;
    const u32 mylen = (u32)lst & ~kListRaw, myoff = (u32)(lst >> 32);
    const bool myraw = ((u32)lst & kListRaw) != 0;
    if (__any_sync(kFull, (u32)lane < m && mylen == 0)) continue;   // a source without a list

    u32 inc = mylen;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o) inc += y;
    }
    if (__shfl_sync(kFull, inc, 31) != len) continue;               // (never) inconsistent lists
    soff[lane] = inc - mylen;
    if (lane == 31) soff[32] = inc;
    if ((u32)lane < m) {
      const Rec<D> r = rec[mysrc];
#pragma unroll
      for (int j = 0; j < D; ++j) tv[lane * D + j] = r.t[j];
    }
    __syncwarp();
    for (u32 k = 0; k < m; ++k) {
      const u32 o = __shfl_sync(kFull, myoff, k), l = __shfl_sync(kFull, mylen, k), so = soff[k];
      for (u32 e = lane; e < l; e += 32) xin[so + e] = L.arena[o + e];
    }
    __syncwarp();
    // raw lists (runs of the spatial sort): index order by counting ranks
    const unsigned rawmask = __ballot_sync(kFull, myraw && (u32)lane < m);
    for (unsigned rm = rawmask; rm; rm &= rm - 1) {
      const u32 k = (u32)__ffs(rm) - 1, so = soff[k], l = soff[k + 1] - so;
      if (l < 2) continue;
      for (u32 e = lane; e < l; e += 32) {
        const u32 x = xin[so + e];
        u32 r = 0;
        for (u32 f = 0; f < l; ++f) r += xin[so + f] < x;
        xout[so + r] = x;
      }
      __syncwarp();
      for (u32 e = lane; e < l; e += 32) xin[so + e] = xout[so + e];
      __syncwarp();
    }
    for (u32 e = lane; e < len; e += 32) {
      u32 k = 0;
      while (soff[k + 1] <= e) ++k;
      const u32 x = xin[e];
      u32 r = e - soff[k];
      for (u32 kk = 0; kk < m; ++kk)
        if (kk != k) r += list_rank(xin + soff[kk], soff[kk + 1] - soff[kk], x);
      xout[r] = x;
      xk[r] = (unsigned char)k;
    }
    __syncwarp();
    // publish the merged list
    unsigned long long at = 0;
    if (lane == 0) at = atomicAdd(L.top, (unsigned long long)len);
    at = __shfl_sync(kFull, at, 0);
    if (at + len <= L.cap) {
      for (u32 e = lane; e < len; e += 32) L.arena[at + e] = xout[e];
      if (lane == 0) L.nxt[ts] = (at << 32) | len;
    }
    const LocVal V{tv, D};
#pragma unroll 1
    for (int j = 0; j < D; ++j) {
      const bool neg = tv[xk[0] * D + j] < 0.0;
      const double sm = warp_fold<D>(0.0, xk, 0, len, V, j);
      if (lane == 0) rs[(i64)ts * D + j] = (neg && sm != 0.0) ? -sm : sm;
    }
    if (lane == 0) L.segdone[q] = 1;
    __syncwarp();
  }
}

constexpr u32 kMergeSrc = 255;   // sources a CTA merge handles (source numbers are bytes)
constexpr u32 kMergeRankSort = 96;   // raw lists up to this length: counting ranks (one warp)
constexpr size_t merge_smem(int d) {
  // in, out (kGatherMax u32 each), source number (kGatherMax u8), per source: offset, slot, list (u32, u32, u64), values
  return (size_t)kGatherMax * 9 + 256 * 16 + 8 + (size_t)256 * d * 8;
}

// One CTA per mixed segment of kGatherWarp < len <= kGatherMax points.
template <int D>
__global__ void __launch_bounds__(256) k_rs_merge(const RsCtl* ctl, const u32* seglen, const u32* outslot,
                                                  const Rec<D>* __restrict__ rec, RsLists L, double* rs,
                                                  const u32* ctalist) {
  extern __shared__ __align__(16) unsigned char msm[];
  double* tv = reinterpret_cast<double*>(msm);                          // 256 x D
  u64* slst = reinterpret_cast<u64*>(msm + (size_t)256 * D * 8);        // 256
  u32* soff = reinterpret_cast<u32*>(slst + 256);                       // 257 (+1 pad)
  u32* ssrc = soff + 258;                                               // 256
  u32* xin = ssrc + 256;                                                // kGatherMax
  u32* xout = xin + kGatherMax;                                         // kGatherMax
  unsigned char* xk = reinterpret_cast<unsigned char*>(xout + kGatherMax);   // kGatherMax
  __shared__ u32 sm_m, sm_ok;
  __shared__ unsigned long long sm_at;
  const u32 nwork = ctl->ncta;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (u32 wi = blockIdx.x; wi < nwork; wi += gridDim.x) {
    const u32 q = ctalist[wi];
    const u32 len = seglen[q];
    const u32 ts = outslot[q];
    __syncthreads();
    if (tid == 0) {
      u32 s = L.shead[ts], m = 0, tot = 0, ok = 1;
      while (s != kRsEmpty && m < kMergeSrc) {
        const u64 lst = L.cur[s];
        ssrc[m] = s;
        slst[m] = lst;
        soff[m] = tot;
        tot += (u32)lst & ~kListRaw;
        ok &= ((u32)lst & ~kListRaw) != 0;
        s = L.snext[s];
        ++m;
      }
      soff[m] = tot;
      sm_m = m;
      sm_ok = ok && s == kRsEmpty && tot == len;
    }
    __syncthreads();
    if (!sm_ok) continue;
    const u32 m = sm_m;
    for (u32 e = tid; e < m * D; e += 256) tv[e] = rec[ssrc[e / D]].t[e % D];
    for (u32 k = w; k < m; k += 8) {
      const u64 lst = slst[k];
      const u32 o = (u32)(lst >> 32), l = (u32)lst & ~kListRaw, so = soff[k];
      for (u32 e = lane; e < l; e += 32) xin[so + e] = L.arena[o + e];
    }
    __syncthreads();
    // raw lists (runs of the spatial sort) are put in index order first: long
    // ones by a block-wide bitonic sort in the output buffer, short ones by
    // counting ranks, a warp each
    for (u32 k = 0; k < m; ++k) {
      const u32 so = soff[k], l = soff[k + 1] - so;
      if (!((u32)slst[k] & kListRaw) || l <= kMergeRankSort) continue;   // block-uniform
      u32 P = 1;
      while (P < l) P <<= 1;
      for (u32 e = tid; e < P; e += 256) xout[e] = e < l ? xin[so + e] : 0xffffffffu;
      __syncthreads();
      for (u32 kk = 2; kk <= P; kk <<= 1)
        for (u32 jj = kk >> 1; jj > 0; jj >>= 1) {
          for (u32 e = tid; e < P; e += 256) {
            const u32 x = e ^ jj;
            if (x > e) {
              const u32 a = xout[e], b = xout[x];
              if ((a > b) == ((e & kk) == 0)) {
                xout[e] = b;
                xout[x] = a;
              }
            }
          }
          __syncthreads();
        }
      for (u32 e = tid; e < l; e += 256) xin[so + e] = xout[e];
      __syncthreads();
    }
    for (u32 k = w; k < m; k += 8) {
      const u32 so = soff[k], l = soff[k + 1] - so;
      if (!((u32)slst[k] & kListRaw) || l > kMergeRankSort || l < 2) continue;
      for (u32 e = lane; e < l; e += 32) {
        const u32 x = xin[so + e];
        u32 r = 0;
        for (u32 f = 0; f < l; ++f) r += xin[so + f] < x;
        xout[so + r] = x;
      }
      __syncwarp();
      for (u32 e = lane; e < l; e += 32) xin[so + e] = xout[so + e];
    }
    __syncthreads();
    for (u32 e = tid; e < len; e += 256) {
      // rank of point e (of source k) among the points of the other sources
      u32 k = 0, hi = m;
      while (hi - k > 1) {
        const u32 md = (k + hi) >> 1;
        if (soff[md] <= e) k = md; else hi = md;
      }
      const u32 x = xin[e];
      u32 r = e - soff[k];
      for (u32 kk = 0; kk < m; ++kk)
        if (kk != k) r += list_rank(xin + soff[kk], soff[kk + 1] - soff[kk], x);
      xout[r] = x;
      xk[r] = (unsigned char)k;
    }
    if (tid == 0) sm_at = atomicAdd(L.top, (unsigned long long)len);
    __syncthreads();
    const unsigned long long at = sm_at;
    if (at + len <= L.cap) {
      for (u32 e = tid; e < len; e += 256) L.arena[at + e] = xout[e];
      if (tid == 0) L.nxt[ts] = (at << 32) | len;
    }
    if (w < D) {
      const LocVal V{tv, D};
      const bool neg = tv[xk[0] * D + w] < 0.0;
      const double sm = warp_fold<D>(0.0, xk, 0, len, V, w);
      if (lane == 0) rs[(i64)ts * D + w] = (neg && sm != 0.0) ? -sm : sm;
    }
    if (tid == 0) L.segdone[q] = 1;
  }
}

// ------------------------------------------------------- sequential model
// GS_SUMS_SEQMODEL: the reference's sequential per-cell sums without the
// point order.  A single-source cell is c copies of one value: the closed
// form, bit for bit.  A mixed target holds c_a copies of each source value
// v_a, interleaved in index order in the reference.  While the accumulator
// stays inside one binade every addition of v_a adds the same number of ulps
// whatever came before (ties aside), so the sum depends on the order only
// through WHICH additions happen before each binade crossing.  The model
// takes a well-mixed order: inside a binade the remaining copies of every
// source are consumed in proportion (one integer multiply-add per source),
// up to the crossing, which is made by single fp64 additions in ascending
// slot order; then the next binade.  (Targets of at most kModelDirect points
// are simply added up, one copy of every source per round.)  Deterministic, a function of the cell
// table only (so independent of how points are split across GPUs), and
// O(sources x binades) per cell instead of O(points).
constexpr u32 kModelSrc = 256;       // sources per target handled in shared memory (3^5 = 243)
constexpr u32 kModelDirect = 96;     // targets up to this many points (<= 32 sources): plain additions
constexpr int kModelWarps = 4;

__device__ __forceinline__ u64 warp_sum_u64(u64 x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}
__device__ __forceinline__ double warp_sum_f64(double x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// One warp folds `m` sources (counts cnt[], magnitudes val[], ascending slot
// order) into the magnitude of their modelled sequential sum.  rem / inc are
// the warp's scratch (m entries each).
__device__ __forceinline__ double model_fold(u32 m, const u32* cnt, const double* val, u32* rem, u64* inc) {
  const int lane = threadIdx.x & 31;
  for (u32 a = lane; a < m; a += 32) rem[a] = cnt[a];
  __syncwarp();
  double s = 0.0;
  for (;;) {
    u64 left = 0;
    for (u32 a = lane; a < m; a += 32) left += rem[a];
    left = warp_sum_u64(left);
    if (left == 0) break;
    bool single = false;          // make single additions this round (first addition / subnormal)
    int be = 0;
    if (s == 0.0) {
      single = true;
    } else {
      const u64 sb = dbits(s);
      be = (int)(sb >> 52);
      if (be <= 1) {
        single = true;
      } else {
        const int ue = be - 1075;
        u64 mi = (sb & ((1ull << 52) - 1)) | (1ull << 52);
        const u64 room = kMaxM - mi;
        double totd = 0.0;
        for (u32 a = lane; a < m; a += 32) {
          u64 ia = 0;
          if (rem[a]) {
            const double x = scale2(val[a], -ue);
            if (x >= 0x1p53) {
              ia = 1ull << 53;                       // crosses at once
            } else {
              const double fl = floor(x);
              const double fr = x - fl;
              ia = (u64)fl + ((fr > 0.5 || (fr == 0.5 && ((u64)fl & 1ull))) ? 1ull : 0ull);
            }
            totd += (double)rem[a] * (double)ia;
          }
          inc[a] = ia;
        }
        totd = warp_sum_f64(totd);
        if (totd == 0.0) break;                       // further additions change nothing
        if (totd <= (double)room * (1.0 - 0x1p-20)) {
          // everything left fits this binade: order-free
          u64 t = 0;
          for (u32 a = lane; a < m; a += 32) t += (u64)rem[a] * inc[a];
          mi += warp_sum_u64(t);
          s = scale2((double)mi, ue);
          break;
        }
        // proportional share of every source up to the crossing
        const double f = (double)room / totd * (1.0 - 0x1p-30);
        u64 tk = 0;
        for (u32 a = lane; a < m; a += 32) {
          u32 take = 0;
          if (rem[a] && inc[a] < (1ull << 53)) {
            const double w = floor(f * (double)rem[a]);
            take = w <= 0.0 ? 0u : (w >= (double)rem[a] ? rem[a] : (u32)w);
          }
          tk += (u64)take * inc[a];
          rem[a] -= take;
          inc[a] = take;                              // (the step is used up; keep the share for an undo)
        }
        tk = warp_sum_u64(tk);
        if (tk > room) {                              // (numerical safety) undo the shares
          for (u32 a = lane; a < m; a += 32) rem[a] += (u32)inc[a];
          tk = 0;
        }
        mi += tk;
        s = scale2((double)mi, ue);
        __syncwarp();
        single = true;                                // the crossing: single additions
      }
    }
    if (single) {
      // single fp64 additions in ascending slot order until the binade changes
      // (one pass at most; the outer loop re-plans)
      __syncwarp();
      for (u32 a = 0; a < m; ++a) {
        if (rem[a] == 0) continue;                    // warp-uniform (shared memory)
        const bool first = s == 0.0;
        s = first ? val[a] : dadd(s, val[a]);
        __syncwarp();
        if (lane == 0) rem[a] -= 1;
        __syncwarp();
        if (first || (int)(dbits(s) >> 52) != be) break;
      }
    }
    __syncwarp();
  }
  return s;
}

// model_fold for up to 32 sources, one per lane (cnt / val lane-private, 0
// beyond the sources): registers and shuffles only.
__device__ __forceinline__ double model_fold32(u32 cnt, double val) {
  const int lane = threadIdx.x & 31;
  u32 rem = cnt;
  double s = 0.0;
  if (__reduce_add_sync(kFull, cnt > kModelDirect ? kModelDirect + 1 : cnt) <= kModelDirect) {
    // a small target: the additions themselves, one copy of every source per
    // round in ascending slot order
    for (;;) {
      unsigned lv = __ballot_sync(kFull, rem > 0);
      if (lv == 0) return s;
      while (lv) {
        const int a = __ffs(lv) - 1;
        lv &= lv - 1;
        const double va = __shfl_sync(kFull, val, a);
        s = s == 0.0 ? va : dadd(s, va);
      }
      rem -= rem > 0;
    }
  }
  for (;;) {
    if (__ballot_sync(kFull, rem > 0) == 0) break;
    bool single = false;
    int be = 0;
    if (s == 0.0) {
      single = true;
    } else {
      const u64 sb = dbits(s);
      be = (int)(sb >> 52);
      if (be <= 1) {
        single = true;
      } else {
        const int ue = be - 1075;
        u64 mi = (sb & ((1ull << 52) - 1)) | (1ull << 52);
        const u64 room = kMaxM - mi;
        u64 ia = 0;
        if (rem) {
          const double x = scale2(val, -ue);
          if (x >= 0x1p53) {
            ia = 1ull << 53;
          } else {
            const double fl = floor(x);
            const double fr = x - fl;
            ia = (u64)fl + ((fr > 0.5 || (fr == 0.5 && ((u64)fl & 1ull))) ? 1ull : 0ull);
          }
        }
        const double totd = warp_sum_f64((double)rem * (double)ia);
        if (totd == 0.0) break;
        if (totd <= (double)room * (1.0 - 0x1p-20)) {
          mi += warp_sum_u64((u64)rem * ia);
          s = scale2((double)mi, ue);
          break;
        }
        const double f = (double)room / totd * (1.0 - 0x1p-30);
        u32 take = 0;
        if (rem && ia < (1ull << 53)) {
          const double w = floor(f * (double)rem);
          take = w <= 0.0 ? 0u : (w >= (double)rem ? rem : (u32)w);
        }
        u64 tk = warp_sum_u64((u64)take * ia);
        if (tk > room) {                              // (numerical safety)
          take = 0;
          tk = 0;
        }
        rem -= take;
        mi += tk;
        s = scale2((double)mi, ue);
        single = true;
      }
    }
    if (single) {
      unsigned lv = __ballot_sync(kFull, rem > 0);
      while (lv) {
        const int a = __ffs(lv) - 1;
        lv &= lv - 1;
        const bool first = s == 0.0;
        const double va = __shfl_sync(kFull, val, a);
        s = first ? va : dadd(s, va);
        if (lane == a) rem -= 1;
        if (first || (int)(dbits(s) >> 52) != be) break;
      }
    }
  }
  return s;
}

template <int D, class Tab>
__global__ void __launch_bounds__(kModelWarps * 32) k_rs_runfold(const RsCtl* ctl, const u32* outslot, Tab cur,
                                                                 const Rec<D>* __restrict__ rec, RsLists L,
                                                                 double* rs) {
  __shared__ u32 s_slot[kModelWarps][kModelSrc];
  __shared__ u32 s_cnt[kModelWarps][kModelSrc];
  __shared__ u32 s_rem[kModelWarps][kModelSrc];
  __shared__ double s_val[kModelWarps][kModelSrc];
  __shared__ u64 s_inc[kModelWarps][kModelSrc];
  const u32 nseg = ctl->nseg;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u32* sl = s_slot[w];
  const i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 q = gw; q < nseg; q += nw) {
    const u32 ts = outslot[q];
    // the sources, ascending by slot (the chain's order is first-come)
    u32 m = 0;
    for (u32 s = L.shead[ts]; s != kRsEmpty; s = L.snext[s]) {
      if (m < kModelSrc && lane == 0) sl[m] = s;
      ++m;
    }
    if (m > kModelSrc) {
      // more sources than the buffers hold (d >= 6 only): source by source,
      // ascending slots found by repeated walks of the chain
      if (lane < D) {
        double acc = 0.0;
        bool neg = false;
        i64 last = -1;
        for (u32 a = 0; a < m; ++a) {
          u32 best = kRsEmpty;
          for (u32 s = L.shead[ts]; s != kRsEmpty; s = L.snext[s])
            if ((i64)s > last && s < best) best = s;
          last = (i64)best;
          const double v = rec[best].t[lane];
          neg |= v < 0.0;
          acc = seqsum_mag_from(acc, fabs(v), cur.ent[best].count);
        }
        rs[(i64)ts * D + lane] = (neg && acc != 0.0) ? -acc : acc;
      }
      __syncwarp();
      continue;
    }
    if (m <= 32) {
      // the common case: one source per lane, registers only
      __syncwarp();
      u32 slot = (u32)lane < m ? sl[lane] : kRsEmpty;
      u32 r = 0;
      for (u32 i = 0; i < m; ++i) r += __shfl_sync(kFull, slot, i) < slot;
      __syncwarp();
      if ((u32)lane < m) sl[r] = slot;
      __syncwarp();
      slot = (u32)lane < m ? sl[lane] : kRsEmpty;
      u32 cnt = 0;
      Rec<D> rr;
#pragma unroll
      for (int j = 0; j < D; ++j) rr.t[j] = 0.0;
      if ((u32)lane < m) {
        cnt = (u32)cur.ent[slot].count;
        rr = rec[slot];
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const bool neg = __any_sync(kFull, rr.t[j] < 0.0);
        const double acc = model_fold32(cnt, fabs(rr.t[j]));
        if (lane == 0) rs[(i64)ts * D + j] = (neg && acc != 0.0) ? -acc : acc;
      }
      __syncwarp();
      continue;
    }
    u32 P = 1;
    while (P < m) P <<= 1;
    for (u32 e = m + lane; e < P; e += 32) sl[e] = kRsEmpty;
    __syncwarp();
    for (u32 k = 2; k <= P; k <<= 1)
      for (u32 jj = k >> 1; jj > 0; jj >>= 1) {
        for (u32 e = lane; e < P; e += 32) {
          const u32 x = e ^ jj;
          if (x > e) {
            const u32 a = sl[e], b = sl[x];
            if ((a > b) == ((e & k) == 0)) {
              sl[e] = b;
              sl[x] = a;
            }
          }
        }
        __syncwarp();
      }
    for (u32 a = lane; a < m; a += 32) s_cnt[w][a] = (u32)cur.ent[sl[a]].count;
#pragma unroll 1
    for (int j = 0; j < D; ++j) {
      bool neg = false;
      for (u32 a = lane; a < m; a += 32) {
        const double v = rec[sl[a]].t[j];
        neg |= v < 0.0;
        s_val[w][a] = fabs(v);
      }
      neg = __any_sync(kFull, neg);
      __syncwarp();
      const double acc = model_fold(m, s_cnt[w], s_val[w], s_rem[w], s_inc[w]);
      if (lane == 0) rs[(i64)ts * D + j] = (neg && acc != 0.0) ? -acc : acc;
      __syncwarp();
    }
  }
}

// Per run of the sorted first iterate: the lowest set bit over its values
// (per axis; atomicMin into low[slot * D + j], initialised to 4096).  A warp
// walks 4096 consecutive positions, 32 at a time, carrying the open run's
// minimum across chunks and flushing only where the cell changes.
template <int D, class Tab>
__global__ void __launch_bounds__(256) k_rs_lowbit(const double* __restrict__ ys, i64 n, GridParams g, Tab tab,
                                                   int* low) {
  const int lane = threadIdx.x & 31;
  const i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  constexpr i64 W = 4096;
  for (i64 w0 = gw * W; w0 < n; w0 += nw * W) {
    u32 cslot = kRsEmpty;
    int cmin[D];
#pragma unroll
    for (int j = 0; j < D; ++j) cmin[j] = 4096;
    for (i64 p0 = w0; p0 < min(n, w0 + W); p0 += 32) {
      const i64 p = p0 + lane;
      u32 slot = kRsEmpty;
      int lb[D];
#pragma unroll
      for (int j = 0; j < D; ++j) lb[j] = 4096;
      if (p < n) {
        double v[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          v[j] = ys[(i64)j * g.ld + p];
          lb[j] = lowbit_exp(v[j]);
        }
        bool inside;
        slot = tab.lookup(pack_key<D>(g, v, inside));
      }
      const unsigned peers = __match_any_sync(kFull, slot);
#pragma unroll
      for (int j = 0; j < D; ++j) lb[j] = __reduce_min_sync(peers, lb[j]);
      const int leader = __ffs(peers) - 1;
      // the group continuing the carried run joins the carry; other groups
      // flush (their run cannot continue past this chunk unless it is the
      // last group, which becomes the carry)
      const u32 last = __shfl_sync(kFull, slot, 31);
      const bool is_carry = slot == cslot;
      const bool is_last = slot == last;
      if (lane == leader && slot != kRsEmpty && !is_carry && !is_last) {
#pragma unroll
        for (int j = 0; j < D; ++j) atomicMin(low + (i64)slot * D + j, lb[j]);
      }
      // update the carry
      if (last != cslot) {
        // flush the old carry (merged with its group in this chunk, if any)
        int m[D];
        const int cl = __ffs(__ballot_sync(kFull, is_carry)) - 1;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const int grp = cl >= 0 ? __shfl_sync(kFull, lb[j], cl) : 4096;
          m[j] = min(cmin[j], grp);
        }
        if (lane == 0 && cslot != kRsEmpty) {
#pragma unroll
          for (int j = 0; j < D; ++j) atomicMin(low + (i64)cslot * D + j, m[j]);
        }
        cslot = last;
#pragma unroll
        for (int j = 0; j < D; ++j) cmin[j] = __shfl_sync(kFull, lb[j], 31);
      } else {
#pragma unroll
        for (int j = 0; j < D; ++j) cmin[j] = min(cmin[j], __shfl_sync(kFull, lb[j], 31));
      }
    }
    if (lane == 0 && cslot != kRsEmpty) {
#pragma unroll
      for (int j = 0; j < D; ++j) atomicMin(low + (i64)cslot * D + j, cmin[j]);
    }
  }
}

// First table: a run's sum provably does not round anywhere when every
// value is a multiple of the ulp of the run's total magnitude (then every
// partial sum -- all of one sign, at most the total -- is representable) and
// of the fixed-point quantum (then the exact table sum is the true sum).
// Every value is a multiple of 2^lowbit[j] (the input's lowest set bit, from
// k_init), so that is a per-run comparison with the exact table sum; those
// runs take it, the others become fold segments.  Also each run's loop slot.
struct LowBits {
  int v[GS_MAXD];
};

template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_rs_first(GridParams g, Tab tab, const u32* runs, const u32* nruns,
                                                       const u32* start, const double* __restrict__ ys,
                                                       bool sorted, bool gather, LowBits lb, u32* rc0, u32* runkey,
                                                       u32* outslot, double* rs, RsCtl* rsc, u32* seglen,
                                                       u32* sstart, u32* send, u32* seglist, u64* runkv,
                                                       const int* lowrun, u64* lst0, bool force_exact) {
  const u32 nr = *nruns;
  const int lane = threadIdx.x & 31;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 w0 = (i64)blockIdx.x * blockDim.x + (threadIdx.x & ~31); w0 < (i64)nr; w0 += stride) {
    const i64 a = w0 + lane;
    const bool valid = a < (i64)nr;
    u32 r = 0, slot = 0, len = 0;
    bool exact = true;
    double S[D];
    if (valid) {
      r = runs[a];
      slot = r;
      if (sorted) {
        double v[D];
#pragma unroll
        for (int j = 0; j < D; ++j) v[j] = ys[(i64)j * g.ld + start[r]];
        bool inside;
        slot = tab.lookup(pack_key<D>(g, v, inside));
      }
      const Entry<D>& e = tab.ent[slot];
      len = (u32)e.count;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        S[j] = i128_to_double((((i128)(i64)e.hi[j]) << 32) + (i128)e.lo[j], -g.qexp[j]);
        const int lbj = lowrun ? lowrun[(i64)slot * D + j] : lb.v[j];
        bool ok = lbj >= -g.qexp[j];
        const double up = fabs(S[j]) * (1.0 + 0x1p-50);
        if (up > 0.0) ok &= lbj >= (int)(dbits(up) >> 52) - 1023 - 52;
        exact &= ok || force_exact;
      }
      rc0[r] = slot;
      // the run's indices: perm[start, start + len), in placement order
      if (lst0) lst0[slot] = len < kListRaw ? (((u64)start[r] << 32) | len | kListRaw) : 0ull;
    }
    const bool seg = valid && !exact;
    const bool big = seg && (!gather || len > kGatherMax);
    // warp-aggregated segment ids and counters
    const unsigned sm = __ballot_sync(kFull, seg);
    u32 m0 = 0;
    if (lane == 0 && sm) m0 = atomicAdd(&rsc->nseg, (u32)__popc(sm));
    m0 = __shfl_sync(kFull, m0, 0);
    const u32 nel = __reduce_add_sync(kFull, big ? len : 0u);
    const unsigned bm = __ballot_sync(kFull, big);
    if (lane == 0 && bm) {
      atomicAdd(&rsc->nelem, nel);
      atomicAdd(&rsc->nbig, (u32)__popc(bm));
    }
    if (!valid) continue;
    if (exact) {
#pragma unroll
      for (int j = 0; j < D; ++j) rs[(i64)slot * D + j] = S[j];
      runkey[r] = kRsEmpty;
      runkv[r] = ~0ull;
    } else {
      const u32 m = m0 + (u32)__popc(sm & ((1u << lane) - 1u));
      outslot[m] = slot;
      seglen[m] = len;
      sstart[m] = 0;
      send[m] = 0;
      runkey[r] = big ? m : kRsEmpty;   // global sort / gathered (the segment is this run)
      runkv[r] = ((u64)kRsEmpty << 32) | (big ? m : kRsEmpty);   // value: the point index
      if (!big) seglist[m] = r;
      atomicMax(&rsc->maxlen, len);
    }
  }
}

// per point: initial slot (unsorted runs; the sorted path has cell0 already)
template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_rs_cell0(const double* __restrict__ y, i64 n, GridParams g, Tab tab,
                                                       u32* cell0) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    double v[D];
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] = y[(i64)j * g.ld + i];
    bool inside;
    cell0[i] = tab.lookup(pack_key<D>(g, v, inside));
  }
}

// final iterate in original point order (AoS): sorted runs share one value
// per run after iteration 0, read at the run's start
__global__ void __launch_bounds__(kThreads) k_iterate_out(const double* __restrict__ y, i64 ld, int d, const u32* cell0,
                                                          const u32* start, i64 n, double* out) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    const i64 p = cell0 ? (i64)start[cell0[i]] : i;
    for (int j = 0; j < d; ++j) out[i * d + j] = y[(i64)j * ld + p];
  }
}

// per-iteration observability: (segments, long segments, their points,
// longest segment, recomputed closed forms)
__global__ void k_rs_stats(const RsCtl* rsc, u32* out) {
  out[0] = rsc->nseg;
  out[1] = rsc->nbig;
  out[2] = rsc->nelem;
  out[3] = rsc->maxlen;
  out[4] = rsc->nsingle;
}

// reset the mixed marks of the targets just folded
__global__ void k_rs_unmark(const u32* outslot, const RsCtl* rsc, u32* mid, u32* shead) {
  const u32 ns = rsc->nseg;
  for (u32 q = blockIdx.x * blockDim.x + threadIdx.x; q < ns; q += gridDim.x * blockDim.x) {
    mid[outslot[q]] = kRsEmpty;
    if (shead) shead[outslot[q]] = kRsEmpty;
  }
}

__global__ void k_rs_set64(unsigned long long* p, unsigned long long v) { *p = v; }

}  // namespace gs
