// gridshift-b200: sm_100a kernels for the MeanShift++ grid shift.
//
// Per iteration t (table buffer b = t & 1, reference modeseek.py:105-111):
//   k_hist   : bin every point (floor(y/h), grid.py:78-85), pack its cell key
//              (grid.py:137-158), and accumulate count + exact fixed-point
//              coordinate sums into the cell table (grid.py:179-190).
//              Warp-aggregated: lanes holding the same key form segments and
//              only the segment head touches the table.
//   k_agg    : per occupied cell, the 3^d neighbourhood count and exact sum
//              (grid.py:230-259), rounded once and divided -> the cell's
//              target mean (modeseek.py:109).  Also clears table b^1 and
//              folds the per-iteration (cells, counts) fingerprint.
//   k_shift  : per point, look up its cell's target, write y', and sum the
//              per-point L2 movement in 128-bit fixed point
//              (modeseek.py:110); the last CTA finishes the reduction and
//              evaluates `movement < eta` (modeseek.py:139) on device.
// Extraction (modeseek.py:229-272): hist of the final iterate, lock-free
// union-find over Chebyshev-adjacent occupied cells, first-appearance
// minimum per component, dense relabel, exact per-component means.
#pragma once

#include "gs_common.cuh"

namespace gs {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;

// ------------------------------------------------------------------ tables

template <int D>
struct DenseTable {
  static constexpr bool kDense = true;
  Entry<D>* ent;
  u32* list;      // occupied slots, in first-touch order
  u32* k;         // occupied count (device)
  __device__ __forceinline__ u64 key_of(u32 s) const { return s; }
  __device__ __forceinline__ bool find(u64 key, u32& s) const {
    s = (u32)key;
    return ent[key].count != 0;
  }
  __device__ __forceinline__ u32 lookup(u64 key) const { return (u32)key; }
  __device__ __forceinline__ u32 insert(u64 key, bool& fresh, int*) const {
    fresh = false;
    return (u32)key;
  }
};

template <int D>
struct HashTable {
  static constexpr bool kDense = false;
  Entry<D>* ent;
  u32* list;
  u32* k;
  u64* keys;      // kEmpty when free
  u64 mask;
  __device__ __forceinline__ u64 key_of(u32 s) const { return keys[s]; }
  __device__ __forceinline__ bool find(u64 key, u32& s) const {
    u64 p = hash_key(key) & mask;
    for (u64 probe = 0; probe <= mask; ++probe) {
      const u64 kk = keys[p];
      if (kk == key) { s = (u32)p; return true; }
      if (kk == kEmpty) return false;
      p = (p + 1) & mask;
    }
    return false;
  }
  __device__ __forceinline__ u32 lookup(u64 key) const {
    u32 s = 0;
    find(key, s);
    return s;
  }
  __device__ __forceinline__ u32 insert(u64 key, bool& fresh, int* err) const {
    u64 p = hash_key(key) & mask;
    for (u64 probe = 0; probe <= mask; ++probe) {
      u64 kk = *(volatile u64*)(keys + p);
      if (kk == kEmpty) {
        kk = atomicCAS(keys + p, kEmpty, key);
        if (kk == kEmpty) { fresh = true; return (u32)p; }
      }
      if (kk == key) { fresh = false; return (u32)p; }
      p = (p + 1) & mask;
    }
    atomicOr(err, kErrTableFull);
    fresh = false;
    return 0xffffffffu;
  }
};

// --------------------------------------------------------------- helpers

// Row sum in numpy's add.reduce order (pairwise_sum: sequential below 8
// elements, an 8-way tree at exactly 8) -- modeseek.py:110 `.sum(axis=1)`.
template <int D>
__device__ __forceinline__ double row_sum(const double* a) {
  if constexpr (D < 8) {
    double r = a[0];
#pragma unroll
    for (int j = 1; j < D; ++j) r = __dadd_rn(r, a[j]);
    return r;
  } else {
    return __dadd_rn(__dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3])),
                     __dadd_rn(__dadd_rn(a[4], a[5]), __dadd_rn(a[6], a[7])));
  }
}

template <int D>
__device__ __forceinline__ u64 cell_fingerprint(const GridParams& g, u64 key, u64 count) {
  u64 x = 0x9E3779B97F4A7C15ull * (u64)(D + 1);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const u64 ext = (j == 0) ? (g.nkeys / g.stride[0]) : (g.stride[j - 1] / g.stride[j]);
    const i64 c = (i64)((key / g.stride[j]) % ext) + g.base[j];
    x = mix64(x ^ (u64)c);
  }
  return mix64(x ^ count);
}

// Pack the cell of one point.  Returns kEmpty if the cell is outside the
// admissible box (flags the error; never happens for valid runs).
template <int D>
__device__ __forceinline__ u64 pack_key(const GridParams& g, const double* v, bool& inside) {
  u64 key = 0;
  inside = true;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const i64 c = (i64)cell_of_fast(v[j], g.h, g.inv_h);
    inside &= (c >= g.lo[j]) & (c <= g.hi[j]);
    key += (u64)(c - g.base[j]) * g.stride[j];
  }
  return inside ? key : kEmpty;
}

// pack_key from the per-axis cells (integer-valued doubles) already taken
template <int D>
__device__ __forceinline__ u64 pack_cells(const GridParams& g, const double* f, bool& inside) {
  u64 key = 0;
  inside = true;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const i64 c = (i64)f[j];
    inside &= (c >= g.lo[j]) & (c <= g.hi[j]);
    key += (u64)(c - g.base[j]) * g.stride[j];
  }
  return inside ? key : kEmpty;
}

__device__ __forceinline__ void add128(u64& hi, u64& lo, u64 ohi, u64 olo) {
  const u64 l = lo + olo;
  hi += ohi + (l < lo ? 1ull : 0ull);
  lo = l;
}

// --------------------------------------------------------------- k_init
// AoS (n, d) input (fp64 or fp32) -> SoA fp64 iterate, plus the per-axis
// cell range, max |coordinate| and input validity (grid.py:42-51, 78-85).

struct InitStats {
  i64 cmin[GS_MAXD];
  i64 cmax[GS_MAXD];
  u64 absmax[GS_MAXD];   // bit pattern of max |x| (non-negative doubles order as ints)
  int flags;
  int pad;
  int lowbit[GS_MAXD];   // min over non-zero values of the exponent of their lowest set bit
};

// exponent of the lowest set bit of |v| (every value is a multiple of 2^it);
// 4096 for zero
__device__ __forceinline__ int lowbit_exp(double v) {
  const u64 b = (u64)__double_as_longlong(v) & ~(1ull << 63);
  if (!b) return 4096;
  const int be = (int)(b >> 52);
  const u64 mant = be ? ((b & ((1ull << 52) - 1)) | (1ull << 52)) : b;
  return (be ? be : 1) - 1075 + __ffsll((long long)mant) - 1;
}

// y == nullptr: statistics only (the sorted path reads x directly).  The
// cell range is taken from the extreme coordinates: fl(v/h) and floor are
// monotonic, so cell(min v) and cell(max v) bound every cell (grid.py:81).
template <int D, typename T>
__global__ void __launch_bounds__(kThreads) k_init_aos(const T* __restrict__ x, double* __restrict__ y,
                                                       i64 n, i64 ld, double h, InitStats* st) {
  const double inv_h = 1.0 / h;
  double vmin[D], vmax[D];
  int low[D];
#pragma unroll
  for (int j = 0; j < D; ++j) { vmin[j] = INFINITY; vmax[j] = -INFINITY; low[j] = 4096; }
  int flags = 0;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double v = (double)x[i * D + j];
      if (y) y[(i64)j * ld + i] = v;
      if (!isfinite(v)) { flags |= kErrNonFinite; continue; }
      vmin[j] = fmin(vmin[j], v);
      vmax[j] = fmax(vmax[j], v);
      low[j] = min(low[j], lowbit_exp(v));
    }
  }
  i64 cmin[D], cmax[D];
  u64 amax[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    cmin[j] = LLONG_MAX; cmax[j] = LLONG_MIN; amax[j] = 0;
    if (vmin[j] <= vmax[j]) {
      const double c0 = cell_of_fast(vmin[j], h, inv_h), c1 = cell_of_fast(vmax[j], h, inv_h);
      if (fabs(c0) >= 4611686018427387904.0 || fabs(c1) >= 4611686018427387904.0) {
        flags |= kErrLattice;
      } else {
        cmin[j] = (i64)c0;
        cmax[j] = (i64)c1;
      }
      amax[j] = (u64)__double_as_longlong(fmax(fabs(vmin[j]), fabs(vmax[j])));
    }
  }
#pragma unroll
  for (int j = 0; j < D; ++j) {
    for (int o = 16; o; o >>= 1) {
      cmin[j] = min(cmin[j], (i64)__shfl_xor_sync(kFull, (unsigned long long)cmin[j], o));
      cmax[j] = max(cmax[j], (i64)__shfl_xor_sync(kFull, (unsigned long long)cmax[j], o));
      amax[j] = max(amax[j], (u64)__shfl_xor_sync(kFull, amax[j], o));
    }
  }
  for (int o = 16; o; o >>= 1) flags |= __shfl_xor_sync(kFull, flags, o);
#pragma unroll
  for (int j = 0; j < D; ++j) low[j] = __reduce_min_sync(kFull, low[j]);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      atomicMin((long long*)&st->cmin[j], (long long)cmin[j]);
      atomicMax((long long*)&st->cmax[j], (long long)cmax[j]);
      atomicMax((unsigned long long*)&st->absmax[j], (unsigned long long)amax[j]);
      atomicMin(&st->lowbit[j], low[j]);
    }
    if (flags) atomicOr(&st->flags, flags);
  }
}

// uint8 image (H, W, 3) -> rgb or rgbxy features (segment.py:82-92), fused.
template <int D>
__global__ void __launch_bounds__(kThreads) k_init_image(const unsigned char* __restrict__ px, double* __restrict__ y,
                                                         i64 n, i64 ld, int width, double scale, double h,
                                                         InitStats* st) {
  i64 cmin[D], cmax[D];
  u64 amax[D];
  int low[D];
#pragma unroll
  for (int j = 0; j < D; ++j) { cmin[j] = LLONG_MAX; cmax[j] = LLONG_MIN; amax[j] = 0; low[j] = 4096; }
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v[D];
    v[0] = (double)px[i * 3 + 0];
    v[1] = (double)px[i * 3 + 1];
    v[2] = (double)px[i * 3 + 2];
    if constexpr (D == 5) {
      const i64 row = i / width;
      const i64 col = i - row * width;
      v[3] = __dmul_rn((double)col, scale);
      v[4] = __dmul_rn((double)row, scale);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      y[(i64)j * ld + i] = v[j];
      const i64 ci = (i64)cell_of(v[j], h);
      cmin[j] = min(cmin[j], ci);
      cmax[j] = max(cmax[j], ci);
      amax[j] = max(amax[j], (u64)__double_as_longlong(fabs(v[j])));
      low[j] = min(low[j], lowbit_exp(v[j]));
    }
  }
#pragma unroll
  for (int j = 0; j < D; ++j) low[j] = __reduce_min_sync(kFull, low[j]);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    for (int o = 16; o; o >>= 1) {
      cmin[j] = min(cmin[j], (i64)__shfl_xor_sync(kFull, (unsigned long long)cmin[j], o));
      cmax[j] = max(cmax[j], (i64)__shfl_xor_sync(kFull, (unsigned long long)cmax[j], o));
      amax[j] = max(amax[j], (u64)__shfl_xor_sync(kFull, amax[j], o));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      atomicMin((long long*)&st->cmin[j], (long long)cmin[j]);
      atomicMax((long long*)&st->cmax[j], (long long)cmax[j]);
      atomicMax((unsigned long long*)&st->absmax[j], (unsigned long long)amax[j]);
      atomicMin(&st->lowbit[j], low[j]);
    }
  }
}

// SoA fp64 -> AoS fp64 (meanshiftpp_step output).
template <int D>
__global__ void k_soa_to_aos(const double* __restrict__ y, double* __restrict__ x, i64 n, i64 ld) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
#pragma unroll
    for (int j = 0; j < D; ++j) x[i * D + j] = y[(i64)j * ld + i];
  }
}

// --------------------------------------------------------------- k_hist

#ifndef GS_HIST_MINB
#define GS_HIST_MINB 3
#endif

// Partial aggregate of a run of points: count and split fixed-point sums.
template <int D>
struct Agg {
  u32 cnt;
  i64 hi[D];
  u64 lo[D];
  __device__ __forceinline__ void zero() {
    cnt = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) { hi[j] = 0; lo[j] = 0; }
  }
  __device__ __forceinline__ void add(const Agg& o) {
    cnt += o.cnt;
#pragma unroll
    for (int j = 0; j < D; ++j) { hi[j] += o.hi[j]; lo[j] += o.lo[j]; }
  }
  __device__ __forceinline__ Agg shfl_up(int off) const {
    Agg r;
    r.cnt = __shfl_up_sync(kFull, cnt, off);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      r.hi[j] = (i64)__shfl_up_sync(kFull, (unsigned long long)hi[j], off);
      r.lo[j] = __shfl_up_sync(kFull, lo[j], off);
    }
    return r;
  }
  // butterfly sum over the warp (every lane ends with the total)
  __device__ __forceinline__ void warp_sum() {
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      cnt += __shfl_xor_sync(kFull, cnt, off);
#pragma unroll
      for (int j = 0; j < D; ++j) {
        hi[j] += (i64)__shfl_xor_sync(kFull, (unsigned long long)hi[j], off);
        lo[j] += __shfl_xor_sync(kFull, lo[j], off);
      }
    }
  }
};

// Flush one finished segment (a run of points with the same cell key).
template <int D, class Tab, bool CountOnly>
__device__ __forceinline__ void flush_segment(const Tab& tab, Ctrl* ctrl, u64 key, const Agg<D>& a) {
  if (key == kEmpty || a.cnt == 0) return;
  bool fresh;
  const u32 s = tab.insert(key, fresh, &ctrl->error);
  if (s == 0xffffffffu) return;
  Entry<D>* e = tab.ent + s;
  // dense tables: no-return atomics (RED); occupancy is read back from the
  // counts where a cell list is needed (k_compact)
  atomicAdd(&e->count, (u64)a.cnt);
  if constexpr (!Tab::kDense) {
    if (fresh) tab.list[atomicAdd(tab.k, 1u)] = s;
  }
  if constexpr (!CountOnly) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      atomicAdd(&e->hi[j], (u64)a.hi[j]);
      atomicAdd(&e->lo[j], a.lo[j]);
    }
  }
}

// Fixed-point item of point m of a lane (count 1), or empty.
template <int D, bool CountOnly>
__device__ __forceinline__ Agg<D> item_of(const GridParams& g, const double* v, bool valid) {
  Agg<D> a;
  a.zero();
  if (valid) {
    a.cnt = 1;
    if constexpr (!CountOnly) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const i64 f = to_fixed(v[j], g.qscale[j]);
        a.hi[j] = f >> 32;
        a.lo[j] = (u64)(f & 0xffffffffll);
      }
    }
  }
  return a;
}

// ---------------------------------------------------------------------------
// Warp reduce-by-key over one 128-point tile (4 consecutive points per lane):
// items are (key[m], src[m]) -> count 1 and the fixed-point image of src[m].
// In-lane sequential aggregation, one segmented inclusive scan of the lane
// tail aggregates, and every finished segment is flushed once by the lane
// holding its successor's head.  The segment still open at the end of the
// tile is carried (ckey, cagg: uniform across lanes) into the next tile of
// the warp's super-tile instead of being flushed -- a run of one cell costs
// one flush per super-tile (hot cells: a mode can hold ~2% of all points,
// and per-tile flushes would serialise thousands of atomics on one L2 line).
// A tile whose 128 items are identical skips the scan.
template <int D, class Tab, bool CountOnly>
__device__ __forceinline__ void rbk_tile(const GridParams& g, const Tab& tab, Ctrl* ctrl, int lane,
                                         const u64 (&key)[4], const double (&src)[4][D],
                                         const bool (&valid)[4], bool tile_uniform, u64& ckey,
                                         Agg<D>& cagg) {
  constexpr int P = 4;
  if (tile_uniform) {
    Agg<D> t = item_of<D, CountOnly>(g, src[0], true);
    t.cnt = 32 * P;
#pragma unroll
    for (int j = 0; j < D; ++j) { t.hi[j] *= 32 * P; t.lo[j] *= 32 * P; }
    if (key[0] == ckey) {
      cagg.add(t);
    } else {
      if (lane == 0) flush_segment<D, Tab, CountOnly>(tab, ctrl, ckey, cagg);
      ckey = key[0];
      cagg = t;
    }
    return;
  }
  u64 prevkey = __shfl_up_sync(kFull, key[P - 1], 1);
  if (lane == 0) prevkey = ckey;
  bool head[P];
  head[0] = key[0] != prevkey;
#pragma unroll
  for (int m = 1; m < P; ++m) head[m] = key[m] != key[m - 1];
  // tail aggregate of this lane (items from its last head on); lane 0
  // starts from the carry when its first item continues it
  Agg<D> x;
  if (lane == 0 && !head[0]) x = cagg; else x.zero();
  bool f = false;
#pragma unroll
  for (int m = 0; m < P; ++m) {
    if (head[m]) { x.zero(); f = true; }
    x.add(item_of<D, CountOnly>(g, src[m], valid[m]));
  }
  // segmented inclusive scan over lanes: x_L = tail_L + (hashead_L ? 0 : x_{L-1})
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const Agg<D> yv = x.shfl_up(off);
    const bool yf = __shfl_up_sync(kFull, f, off);
    if (lane >= off && !f) { x.add(yv); f = yf; }
  }
  Agg<D> acc = x.shfl_up(1);   // open segment carried in from the lanes before
  if (lane == 0) acc = cagg;
#pragma unroll
  for (int m = 0; m < P; ++m) {
    const Agg<D> itm = item_of<D, CountOnly>(g, src[m], valid[m]);
    if (head[m]) {
      flush_segment<D, Tab, CountOnly>(tab, ctrl, m ? key[m - 1] : prevkey, acc);
      acc = itm;
    } else {
      acc.add(itm);
    }
  }
  // lane 31's open segment becomes the carry
  ckey = __shfl_sync(kFull, key[P - 1], 31);
  cagg.cnt = __shfl_sync(kFull, acc.cnt, 31);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    cagg.hi[j] = (i64)__shfl_sync(kFull, (unsigned long long)acc.hi[j], 31);
    cagg.lo[j] = __shfl_sync(kFull, acc.lo[j], 31);
  }
}

#ifndef GS_HIST_S
#define GS_HIST_S 8
#endif
constexpr int kSuper = GS_HIST_S;   // tiles per warp super-tile
#ifndef GS_HIST_PF
#define GS_HIST_PF 1
#endif

// Load a lane's 4 consecutive points of tile starting at i0 (SoA, 16-byte
// vector loads) and classify: `uni` = the lane's 4 points are bitwise
// identical (and in range), return = every lane of the tile holds the same
// point (the tile is uniform).
template <int D>
__device__ __forceinline__ bool load_quad(const double* __restrict__ y, const GridParams& g, i64 i0, i64 n,
                                          double (&v)[4][D], bool& uni) {
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double2* src = reinterpret_cast<const double2*>(y + (i64)j * g.ld + i0);
    const double2 a = __ldcs(src), b = __ldcs(src + 1);
    v[0][j] = a.x; v[1][j] = a.y; v[2][j] = b.x; v[3][j] = b.y;
  }
  uni = i0 + 3 < n;
#pragma unroll
  for (int m = 1; m < 4; ++m)
#pragma unroll
    for (int j = 0; j < D; ++j) uni &= __double_as_longlong(v[m][j]) == __double_as_longlong(v[0][j]);
  bool same = uni;
#pragma unroll
  for (int j = 0; j < D; ++j)
    same &= __shfl_sync(kFull, __double_as_longlong(v[0][j]), 0) == __double_as_longlong(v[0][j]);
  return __all_sync(kFull, same);
}

// Histogram of one iterate into a clean table (first iteration, extraction
// of a user-given point set, table dumps; the loop derives later tables).
// Warps take strided super-tiles of kSuper consecutive 128-point tiles, so
// the grid streams through a narrow window of memory.
// Fresh: the input points of a run (first table) -- identical points are not
// expected, so the per-quad / per-tile bitwise-identity tests are skipped.
// Grouped: the points of each cell are contiguous (the output of the spatial
// sort), so a tile is key-uniform iff its first and last points share a cell:
// two keys per tile instead of one per point.
template <int D, class Tab, bool CountOnly = false, bool Fresh = false, bool Grouped = false>
__global__ void __launch_bounds__(kThreads, (D <= 3 ? GS_HIST_MINB : 2)) k_hist(const double* __restrict__ y, i64 n, GridParams g,
                                                   Tab tab, Ctrl* ctrl, int check_done) {
  if (check_done && *(volatile int*)&ctrl->done) return;
  constexpr int P = 4;
  constexpr int TILE = 32 * P;
  const int lane = threadIdx.x & 31;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  const i64 ntiles = (n + TILE - 1) / TILE;
  const i64 nsuper = (ntiles + kSuper - 1) / kSuper;
  for (i64 sup = warp; sup < nsuper; sup += nwarps) {
    u64 ckey = kEmpty;
    Agg<D> cagg;
    cagg.zero();
    // dist: the carry is spread over the lanes (its value is the sum of the
    // lanes' cagg) -- key-uniform tiles (all 128 points in the open cell, the
    // common case on a cell-sorted iterate) add into it lane-privately, with
    // no shuffles; it is folded back before anything reads it
    bool dist = false;
    const i64 t_end = min(ntiles, (sup + 1) * kSuper);
    for (i64 tile = sup * kSuper; tile < t_end; ++tile) {
      const i64 i0 = tile * TILE + P * lane;
      if (GS_HIST_PF > 0 && tile + GS_HIST_PF < t_end) {
        // L2 prefetch GS_HIST_PF tiles ahead: the next loads of this warp
        // hit L2 instead of waiting the full HBM latency
#pragma unroll
        for (int j = 0; j < D; ++j)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(y + (i64)j * g.ld + i0 + GS_HIST_PF * TILE));
      }
      double v[P][D];
      bool uni = false, tu = false;
      if constexpr (Fresh) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double2* src = reinterpret_cast<const double2*>(y + (i64)j * g.ld + i0);
          const double2 a = __ldcs(src), b = __ldcs(src + 1);
          v[0][j] = a.x; v[1][j] = a.y; v[2][j] = b.x; v[3][j] = b.y;
        }
      } else {
        tu = load_quad<D>(y, g, i0, n, v, uni);
      }
      bool valid[P];
#pragma unroll
      for (int m = 0; m < P; ++m) valid[m] = i0 + m < n;
      if (Grouped && !tu) {
        u64 kend = kEmpty;
        if (lane == 0 || lane == 31) {
          double w[D];
#pragma unroll
          for (int j = 0; j < D; ++j) w[j] = lane == 0 ? v[0][j] : v[P - 1][j];
          bool inside;
          kend = pack_key<D>(g, w, inside);
        }
        const u64 k0 = __shfl_sync(kFull, kend, 0);
        const bool full_tile = __shfl_sync(kFull, (int)valid[P - 1], 31);
        if (full_tile && k0 != kEmpty && k0 == __shfl_sync(kFull, kend, 31)) {
          if (k0 != ckey) {
            if (dist) cagg.warp_sum();
            if (lane == 0) flush_segment<D, Tab, CountOnly>(tab, ctrl, ckey, cagg);
            ckey = k0;
            cagg.zero();
          } else if (!dist && lane) {
            cagg.zero();   // lane 0 keeps the (uniform) carry
          }
          dist = true;
#pragma unroll
          for (int m = 0; m < P; ++m) cagg.add(item_of<D, CountOnly>(g, v[m], true));
          continue;
        }
      } else if (!tu) {
        // key-uniform tile (all 128 points in one cell, the common case on a
        // cell-sorted iterate): decided on the per-axis floors, the key is
        // packed once; the points add lane-privately into the spread carry
        double f0[D];
#pragma unroll
        for (int j = 0; j < D; ++j) f0[j] = cell_of_fast(v[0][j], g.h, g.inv_h);
        bool ku = valid[P - 1];
        if (!uni) {
#pragma unroll
          for (int m = 1; m < P; ++m)
#pragma unroll
            for (int j = 0; j < D; ++j) ku &= cell_of_fast(v[m][j], g.h, g.inv_h) == f0[j];
        }
#pragma unroll
        for (int j = 0; j < D; ++j) ku &= __shfl_sync(kFull, f0[j], 0) == f0[j];
        bool inside = false;
        const u64 k0 = pack_cells<D>(g, f0, inside);
        if (__all_sync(kFull, ku) && inside) {   // inside is warp-uniform here
          if (k0 != ckey) {
            if (dist) cagg.warp_sum();
            if (lane == 0) flush_segment<D, Tab, CountOnly>(tab, ctrl, ckey, cagg);
            ckey = k0;
            cagg.zero();
          } else if (!dist && lane) {
            cagg.zero();   // lane 0 keeps the (uniform) carry
          }
          dist = true;
#pragma unroll
          for (int m = 0; m < P; ++m) cagg.add(item_of<D, CountOnly>(g, v[m], true));
          continue;
        }
      }
      u64 key[P];
      if (uni) {
        bool inside;
        key[0] = pack_key<D>(g, v[0], inside);
        if (!inside) atomicOr(&ctrl->error, kErrOutOfBox);
#pragma unroll
        for (int m = 1; m < P; ++m) key[m] = key[0];
      } else {
#pragma unroll
        for (int m = 0; m < P; ++m) {
          key[m] = kEmpty;
          if (valid[m]) {
            bool inside;
            key[m] = pack_key<D>(g, v[m], inside);
            if (!inside) atomicOr(&ctrl->error, kErrOutOfBox);
          }
        }
      }
      if (dist) { cagg.warp_sum(); dist = false; }
      rbk_tile<D, Tab, CountOnly>(g, tab, ctrl, lane, key, v, valid, tu, ckey, cagg);
    }
    if (dist) cagg.warp_sum();
    if (lane == 0) flush_segment<D, Tab, CountOnly>(tab, ctrl, ckey, cagg);
  }
}

// Cell record written by k_agg: the target (the cell's 3^d-neighbourhood
// mean, D doubles) followed by the packed key of the target's own cell.
template <int D>
struct Rec {
  double t[D];
  u64 key;
};

// Movement of one point, as a 128-bit fixed-point increment.
template <int D>
__device__ __forceinline__ u128 move_fixed(const GridParams& g, const double* t, const double* v) {
  double sq[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double dlt = __dsub_rn(t[j], v[j]);
    sq[j] = __dmul_rn(dlt, dlt);
  }
  return norm_to_fixed(__dsqrt_rn(row_sum<D>(sq)), g.movement_exp);
}

template <int D, class Tab>
__device__ __forceinline__ const Rec<D>& lookup_rec(const GridParams& g, const Tab& tab, const Rec<D>* rec,
                                                    const double* v, Ctrl* ctrl) {
  bool inside;
  const u64 key = pack_key<D>(g, v, inside);
  u32 s = 0;
  if constexpr (Tab::kDense) {
    if (inside) s = (u32)key; else atomicOr(&ctrl->error, kErrMissing);
  } else {
    if (!inside || !tab.find(key, s)) { atomicOr(&ctrl->error, kErrMissing); s = 0; }
  }
  return rec[s];
}

// One quad: look up the cell records, produce y' (out), accumulate the exact
// movement.  `in` holds points 4q..4q+3 per axis as two double2.
// Returns kQuadMixed (outputs to compare per pair), kQuadStill (uniform
// quad already at its target: nothing to store) or kQuadMoved (uniform quad
// that moved: every coordinate changes).
constexpr int kQuadMixed = 0, kQuadStill = 1, kQuadMoved = 2;

template <int D, class Tab>
__device__ __forceinline__ int shift_quad(const GridParams& g, const Tab& tab, const Rec<D>* __restrict__ rec,
                                          Ctrl* ctrl, const double2 (&in)[D][2], i64 q, i64 n,
                                          double (&out)[4][D], u64& ahi, u64& alo) {
  bool uni = 4 * q + 3 < n;
#pragma unroll
  for (int j = 0; j < D; ++j)
    uni &= (__double_as_longlong(in[j][0].x) == __double_as_longlong(in[j][0].y)) &
           (__double_as_longlong(in[j][0].x) == __double_as_longlong(in[j][1].x)) &
           (__double_as_longlong(in[j][0].x) == __double_as_longlong(in[j][1].y));
  if (uni) {
    double v[D];
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] = in[j][0].x;
    const Rec<D>& r = lookup_rec<D>(g, tab, rec, v, ctrl);
    bool still = true;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      out[0][j] = r.t[j];
      still &= __double_as_longlong(out[0][j]) == __double_as_longlong(v[j]);
    }
    if (!still) {   // a quad at its target moves by exactly 0
      const u128 f = move_fixed<D>(g, out[0], v) << 2;
      add128(ahi, alo, (u64)(f >> 64), (u64)f);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) out[1][j] = out[2][j] = out[3][j] = out[0][j];
    return still ? kQuadStill : kQuadMoved;
  } else {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      double v[D];
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = (m & 1) ? in[j][m >> 1].y : in[j][m >> 1].x;
      if (4 * q + m < n) {
        const Rec<D>& r = lookup_rec<D>(g, tab, rec, v, ctrl);
#pragma unroll
        for (int j = 0; j < D; ++j) out[m][j] = r.t[j];
        const u128 f = move_fixed<D>(g, out[m], v);
        add128(ahi, alo, (u64)(f >> 64), (u64)f);
      } else {
#pragma unroll
        for (int j = 0; j < D; ++j) out[m][j] = v[j];
      }
    }
  }
  return kQuadMixed;
}

// Store y' of a quad into yo; with an in-place iterate, 16-byte pairs whose
// coordinates are bitwise unchanged are not rewritten.
template <int D>
__device__ __forceinline__ void store_quad(double* yo, i64 ld, i64 q, bool inplace, const double2 (&in)[D][2],
                                           const double (&out)[4][D], u32& nst, int kind = kQuadMixed) {
  if (inplace && kind == kQuadStill) return;
  if (kind == kQuadMoved || !inplace) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double2* dst = reinterpret_cast<double2*>(yo + (i64)j * ld) + 2 * q;
      __stcs(dst, make_double2(out[0][j], out[1][j]));
      __stcs(dst + 1, make_double2(out[2][j], out[3][j]));
    }
    nst += 2 * D;
    return;
  }
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double2* dst = reinterpret_cast<double2*>(yo + (i64)j * ld) + 2 * q;
    const bool same0 = inplace && __double_as_longlong(out[0][j]) == __double_as_longlong(in[j][0].x) &&
                       __double_as_longlong(out[1][j]) == __double_as_longlong(in[j][0].y);
    const bool same1 = inplace && __double_as_longlong(out[2][j]) == __double_as_longlong(in[j][1].x) &&
                       __double_as_longlong(out[3][j]) == __double_as_longlong(in[j][1].y);
    if (!same0) { __stcs(dst, make_double2(out[0][j], out[1][j])); ++nst; }
    if (!same1) { __stcs(dst + 1, make_double2(out[2][j], out[3][j])); ++nst; }
  }
}

// Block reduction of the 128-bit movement and the store count; the last CTA
// finishes: movement < eta (modeseek.py:139) on device, or the 4 limbs of
// this rank's exact total for a sharded run.
template <int D>
__device__ __forceinline__ void finish_movement(const GridParams& g, Ctrl* ctrl, u64* partials, double* mv_hist,
                                                int t, double eta, u64* limbs, u64* wbytes, u64 ahi, u64 alo,
                                                u32 nst) {
  const int lane = threadIdx.x & 31;
  for (int off = 16; off; off >>= 1) {
    const u64 oh = __shfl_xor_sync(kFull, ahi, off);
    const u64 ol = __shfl_xor_sync(kFull, alo, off);
    add128(ahi, alo, oh, ol);
  }
  nst = __reduce_add_sync(kFull, nst);
  __shared__ u64 sh[32][2];   // up to 1024 threads
  __shared__ u32 shn[32];
  __shared__ bool last;
  const int w = threadIdx.x >> 5;
  if (lane == 0) { sh[w][0] = ahi; sh[w][1] = alo; shn[w] = nst; }
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 bh = 0, bl = 0, bn = 0;
    for (int qq = 0; qq < (int)(blockDim.x >> 5); ++qq) { add128(bh, bl, sh[qq][0], sh[qq][1]); bn += shn[qq]; }
    if (wbytes && bn) atomicAdd((unsigned long long*)wbytes, (unsigned long long)(16 * bn));
    partials[2 * blockIdx.x] = bh;
    partials[2 * blockIdx.x + 1] = bl;
    __threadfence();
    const u32 ticket = atomicAdd(&ctrl->blocks_done, 1u);
    last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  u64 th = 0, tl = 0;
  for (u32 b = threadIdx.x; b < gridDim.x; b += blockDim.x)
    add128(th, tl, __ldcg(partials + 2 * b), __ldcg(partials + 2 * b + 1));
  for (int off = 16; off; off >>= 1) {
    const u64 oh = __shfl_xor_sync(kFull, th, off);
    const u64 ol = __shfl_xor_sync(kFull, tl, off);
    add128(th, tl, oh, ol);
  }
  __syncthreads();
  if (lane == 0) { sh[w][0] = th; sh[w][1] = tl; }
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 bh = 0, bl = 0;
    for (int qq = 0; qq < (int)(blockDim.x >> 5); ++qq) add128(bh, bl, sh[qq][0], sh[qq][1]);
    ctrl->blocks_done = 0;
    if (limbs) {
      // sharded run: this rank's exact total as 32-bit limbs, summed across
      // ranks by an integer all-reduce, then k_converge
      limbs[0] = bl & 0xffffffffull;
      limbs[1] = bl >> 32;
      limbs[2] = bh & 0xffffffffull;
      limbs[3] = bh >> 32;
      return;
    }
    const double mv = u128_to_double((((u128)bh) << 64) | (u128)bl, g.movement_exp - 96);
    mv_hist[t] = mv;
    ctrl->iters = t + 1;
    if (mv < eta) ctrl->done = t + 1;   // stamped: the run stopped after iteration t
  }
}

// Shift of iteration t (modeseek.py:109-110): per 4-point quad (two 16-byte
// vector loads per SoA axis) look up the cell record, write y' = target,
// accumulate the per-point L2 movement in 128-bit fixed point.  Quads of
// bitwise-identical points (every cell-sorted run after iteration 0) share
// one lookup and one norm (exact: identical inputs, movement scaled by 4 in
// fixed point).  The iterate is updated IN PLACE (y == yo is allowed: each
// quad is read and written by one thread only, lookups go through the cell
// records), and a 16-byte store whose two coordinates are bitwise unchanged
// is elided -- once clusters settle most points sit at their cell's target,
// so converged iterations stream mostly reads.  `wbytes` counts the bytes
// actually stored (per-iteration trace, for the roofline accounting).
// Register-prefetched variant (any table); dense tables use k_shift_tma.
template <int D, class Tab>
__global__ void __launch_bounds__(kThreads, 2) k_shift(const double* y, double* yo, i64 n,
                                                       GridParams g, Tab tab, const Rec<D>* __restrict__ rec,
                                                       Ctrl* ctrl, u64* partials, double* mv_hist, int t,
                                                       double eta, u64* limbs, u64* wbytes) {
  if (*(volatile int*)&ctrl->done) return;
  u64 ahi = 0, alo = 0;
  u32 nst = 0;   // 16-byte stores issued
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const i64 nquads = (n + 3) >> 2;
  // software pipelined: the next quad's loads are in flight while this one
  // is looked up and compared
  i64 q = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  double2 nx[D][2];
  if (q < nquads) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double2* src = reinterpret_cast<const double2*>(y + (i64)j * g.ld) + 2 * q;
      nx[j][0] = __ldcs(src);
      nx[j][1] = __ldcs(src + 1);
    }
  }
  for (; q < nquads; q += stride) {
    double2 in[D][2];
#pragma unroll
    for (int j = 0; j < D; ++j) { in[j][0] = nx[j][0]; in[j][1] = nx[j][1]; }
    if (q + stride < nquads) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double2* src = reinterpret_cast<const double2*>(y + (i64)j * g.ld) + 2 * (q + stride);
        nx[j][0] = __ldcs(src);
        nx[j][1] = __ldcs(src + 1);
      }
    }
    double out[4][D];
    const int kind = shift_quad<D, Tab>(g, tab, rec, ctrl, in, q, n, out, ahi, alo);
    store_quad<D>(yo, g.ld, q, y == yo, in, out, nst, kind);
  }
  finish_movement<D>(g, ctrl, partials, mv_hist, t, eta, limbs, wbytes, ahi, alo, nst);
}

// ---- TMA-pipelined shift (dense tables, in-place iterate).  A persistent
// CTA of T threads walks tiles of 4*T points; one thread keeps kShiftStages tiles
// in flight with 1-D bulk copies (cp.async.bulk, completion on an mbarrier),
// so the read stream needs no registers and no per-thread latency hiding.
#ifndef GS_SHIFT_STAGES
#define GS_SHIFT_STAGES 2
#endif
constexpr int kShiftStages = GS_SHIFT_STAGES;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int D, int T = kThreads>
constexpr size_t shift_tma_smem() {
  return (size_t)kShiftStages * D * 4 * T * sizeof(double);
}

// (Dense tables do not read `tab`: the key is the slot.  Hash tables probe it;
// their 4- and 5-axis quads need more registers.)
template <int D, int T, class Tab>
__global__ void __maxnreg__(D <= 3 ? 96 : 128) k_shift_tma(double* y, i64 n, GridParams g, Tab tab,
                                                           const Rec<D>* __restrict__ rec, Ctrl* ctrl,
                                                           u64* partials, double* mv_hist, int t, double eta,
                                                           u64* limbs, u64* wbytes) {
  if (*(volatile int*)&ctrl->done) return;
  constexpr int kShiftTilePts = 4 * T;
  extern __shared__ __align__(128) double tiles[];   // [stage][axis][kShiftTilePts]
  __shared__ __align__(8) u64 full[kShiftStages];
  const i64 ntiles = (n + kShiftTilePts - 1) / kShiftTilePts;
  const i64 G = gridDim.x;
  const i64 mine = (ntiles > (i64)blockIdx.x) ? (ntiles - (i64)blockIdx.x + G - 1) / G : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kShiftStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](i64 k) {
    const i64 p0 = ((i64)blockIdx.x + k * G) * kShiftTilePts;
    const i64 cnt = min((i64)kShiftTilePts, n - p0);
    const u32 bytes = (u32)(((cnt + 1) & ~1ll) * (i64)sizeof(double));   // 16-byte multiple (ld pads)
    const int s = (int)(k % kShiftStages);
    mbar_expect_tx(&full[s], bytes * D);
#pragma unroll
    for (int j = 0; j < D; ++j)
      bulk_g2s(tiles + ((size_t)s * D + j) * kShiftTilePts, y + (i64)j * g.ld + p0, bytes, &full[s]);
  };
  if (threadIdx.x == 0)
    for (i64 k = 0; k < min((i64)kShiftStages, mine); ++k) issue(k);
  u64 ahi = 0, alo = 0;
  u32 nst = 0;
  for (i64 k = 0; k < mine; ++k) {
    const int s = (int)(k % kShiftStages);
    mbar_wait(&full[s], (u32)((k / kShiftStages) & 1));
    const i64 q = (((i64)blockIdx.x + k * G) * kShiftTilePts >> 2) + threadIdx.x;
    if (4 * q < n) {
      double2 in[D][2];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double2* src = reinterpret_cast<const double2*>(tiles + ((size_t)s * D + j) * kShiftTilePts) +
                             2 * threadIdx.x;
        in[j][0] = src[0];
        in[j][1] = src[1];
      }
      double out[4][D];
      const int kind = shift_quad<D, Tab>(g, tab, rec, ctrl, in, q, n, out, ahi, alo);
      store_quad<D>(y, g.ld, q, true, in, out, nst, kind);
    }
    __syncthreads();   // stage s consumed: refill it
    if (threadIdx.x == 0 && k + kShiftStages < mine) issue(k + kShiftStages);
  }
  finish_movement<D>(g, ctrl, partials, mv_hist, t, eta, limbs, wbytes, ahi, alo, nst);
}

// Collapsed formulation: after iteration 0 all points of a run
// (initial cell) share one position, so iterations t >= 1 move one position
// per run.  runpos: SoA (D x R) positions, runcnt: points per run.  The
// movement is count * fixed(norm) per run -- the same exact integer as the
// per-point sum, so every result is bit-identical to the per-point path.
template <int D>
__global__ void k_runs_gather(const double* __restrict__ y, i64 ld, const u32* runs, const u32* nruns,
                              const u32* start, const u32* end, double* runpos, u32* runcnt, i64 rld) {
  const u32 R = *nruns;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride) {
    const u32 s0 = runs[r];
    const u32 p = start[s0];
#pragma unroll
    for (int j = 0; j < D; ++j) runpos[(i64)j * rld + r] = y[(i64)j * ld + p];
    runcnt[r] = end[s0] - p;
  }
}

template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_run_shift(double* __restrict__ runpos, const u32* __restrict__ runcnt,
                                                        const u32* nruns, i64 rld, GridParams g, Tab tab,
                                                        const Rec<D>* __restrict__ rec, Ctrl* ctrl, u64* partials,
                                                        double* mv_hist, int t, double eta) {
  if (*(volatile int*)&ctrl->done) return;
  const u32 R = *nruns;
  u64 ahi = 0, alo = 0;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < R; r += stride) {
    double v[D], o[D];
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] = runpos[(i64)j * rld + r];
    const Rec<D>& rr = lookup_rec<D>(g, tab, rec, v, ctrl);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      o[j] = rr.t[j];
      runpos[(i64)j * rld + r] = o[j];
    }
    const u128 f = move_fixed<D>(g, o, v) * (u128)runcnt[r];
    add128(ahi, alo, (u64)(f >> 64), (u64)f);
  }
  const int lane = threadIdx.x & 31;
  for (int off = 16; off; off >>= 1) {
    const u64 oh = __shfl_xor_sync(kFull, ahi, off);
    const u64 ol = __shfl_xor_sync(kFull, alo, off);
    add128(ahi, alo, oh, ol);
  }
  __shared__ u64 sh[kThreads / 32][2];
  __shared__ bool last;
  const int w = threadIdx.x >> 5;
  if (lane == 0) { sh[w][0] = ahi; sh[w][1] = alo; }
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 bh = 0, bl = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) add128(bh, bl, sh[q][0], sh[q][1]);
    partials[2 * blockIdx.x] = bh;
    partials[2 * blockIdx.x + 1] = bl;
    __threadfence();
    last = (atomicAdd(&ctrl->blocks_done, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  u64 th = 0, tl = 0;
  for (u32 b = threadIdx.x; b < gridDim.x; b += blockDim.x)
    add128(th, tl, __ldcg(partials + 2 * b), __ldcg(partials + 2 * b + 1));
  for (int off = 16; off; off >>= 1) {
    const u64 oh = __shfl_xor_sync(kFull, th, off);
    const u64 ol = __shfl_xor_sync(kFull, tl, off);
    add128(th, tl, oh, ol);
  }
  __syncthreads();
  if (lane == 0) { sh[w][0] = th; sh[w][1] = tl; }
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 bh = 0, bl = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) add128(bh, bl, sh[q][0], sh[q][1]);
    ctrl->blocks_done = 0;
    const double mv = u128_to_double((((u128)bh) << 64) | (u128)bl, g.movement_exp - 96);
    mv_hist[t] = mv;
    ctrl->iters = t + 1;
    if (mv < eta) ctrl->done = t + 1;   // stamped: the run stopped after iteration t
  }
}

// Sharded run: global movement from the all-reduced limbs (exact).
__global__ void k_converge(const u64* limbs, GridParams g, Ctrl* ctrl, double* mv_hist, int t, double eta) {
  if (*(volatile int*)&ctrl->done) return;
  const u128 tot = (u128)limbs[0] + ((u128)limbs[1] << 32) + ((u128)limbs[2] << 64) + ((u128)limbs[3] << 96);
  const double mv = u128_to_double(tot, g.movement_exp - 96);
  mv_hist[t] = mv;
  ctrl->iters = t + 1;
  if (mv < eta) ctrl->done = t + 1;   // stamped: the run stopped after iteration t
}

// Sharded run: per-root first-appearance minima (global indices) for a MIN
// all-reduce; non-roots stay at the sentinel.
template <int D, class Tab>
__global__ void k_export_minima(Tab tab, const u32* kp, const u32* par, const u32* first, long long* minima) {
  const u32 k = *kp;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < k; a += stride) {
    const u32 s = tab.list[a];
    if (par[s] == s && first[s] != 0xffffffffu) minima[s] = (long long)first[s];
  }
}

template <int D, class Tab>
__global__ void k_import_minima(Tab tab, const u32* kp, const u32* par, u32* first, const long long* minima) {
  const u32 k = *kp;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < k; a += stride) {
    const u32 s = tab.list[a];
    if (par[s] == s) first[s] = (u32)minima[s];
  }
}

// d >= 4 (81 or more neighbours): one warp per occupied cell, the lanes
// split the 3^d offsets (independent probes in flight), then a warp
// reduction of the exact 128-bit sums.
template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_agg_warp(GridParams g, Tab tab, Tab prev, Rec<D>* __restrict__ rec,
                                                       Ctrl* ctrl, int cur, u64* fp_out, u32* k_out, int t,
                                                       const double* __restrict__ rs = nullptr) {
  if (block_stopped_before(ctrl, t)) return;
  constexpr int M = (D == 1) ? 3 : (D == 2) ? 9 : (D == 3) ? 27 : (D == 4) ? 81 :
                    (D == 5) ? 243 : (D == 6) ? 729 : (D == 7) ? 2187 : 6561;
  // reference order: the lanes fetch 32 neighbours at a time into shared
  // memory, lanes j < D then add axis j sequentially in offset order
  __shared__ double nb_s[kThreads / 32][32][D];
  const int lane = threadIdx.x & 31;
  const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  {
    const u32 kp = ctrl->k[cur ^ 1];
    for (i64 a = tid; a < kp; a += stride) {
      const u32 s = prev.list[a];
      Entry<D>* e = prev.ent + s;
      e->count = 0;
#pragma unroll
      for (int j = 0; j < D; ++j) { e->hi[j] = 0; e->lo[j] = 0; }
      if constexpr (!Tab::kDense) prev.keys[s] = kEmpty;
    }
  }
  const i64 warp = tid >> 5;
  const i64 nwarps = stride >> 5;
  const u32 k = ctrl->k[cur];
  u64 fp = 0;
  u32 kc = 0;
  for (i64 a = warp; a < k; a += nwarps) {
    const u32 s = tab.list[a];
    const u64 key = tab.key_of(s);
    u64 cnt = 0;
    u64 sh[D], sl[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { sh[j] = 0; sl[j] = 0; }
    double rsum = 0.0;   // lane j < D: axis j in reference order
    const int wl = threadIdx.x >> 5;
    for (int o0 = 0; o0 < M; o0 += 32) {
      const int o = o0 + lane;
      int r = o;
      i64 delta = 0;
#pragma unroll
      for (int j = D - 1; j >= 0; --j) {
        delta += (i64)((r % 3) - 1) * (i64)g.stride[j];
        r /= 3;
      }
      u32 ns;
      const bool hit = o < M && tab.find(key + (u64)delta, ns);
      if (hit) {
        const Entry<D>& e = tab.ent[ns];
        cnt += e.count;
        if (rs) {
#pragma unroll
          for (int j = 0; j < D; ++j) nb_s[wl][lane][j] = rs[(i64)ns * D + j];
        } else {
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const i128 v = (((i128)(i64)e.hi[j]) << 32) + (i128)e.lo[j];
            add128(sh[j], sl[j], (u64)((u128)v >> 64), (u64)v);
          }
        }
      }
      if (rs) {
        const unsigned hm = __ballot_sync(kFull, hit);
        __syncwarp();
        if (lane < D) {
          unsigned mm = hm;
          while (mm) {
            const int q = __ffs(mm) - 1;
            mm &= mm - 1;
            rsum = __dadd_rn(rsum, nb_s[wl][q][lane]);
          }
        }
        __syncwarp();
      }
    }
    for (int off = 16; off; off >>= 1) {
      cnt += __shfl_xor_sync(kFull, cnt, off);
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const u64 oh = __shfl_xor_sync(kFull, sh[j], off);
        const u64 ol = __shfl_xor_sync(kFull, sl[j], off);
        add128(sh[j], sl[j], oh, ol);
      }
    }
    double rsv[D];
#pragma unroll
    for (int j = 0; j < D; ++j) rsv[j] = __shfl_sync(kFull, rsum, j);
    if (lane == 0) {
      Rec<D> rr;
      const double c = (double)cnt;
#pragma unroll
      for (int j = 0; j < D; ++j)
        rr.t[j] = rs ? __ddiv_rn(rsv[j], c)
                     : __ddiv_rn(i128_to_double((i128)((((u128)sh[j]) << 64) | (u128)sl[j]), -g.qexp[j]), c);
      bool inside;
      rr.key = pack_key<D>(g, rr.t, inside);
      if (!inside) atomicOr(&ctrl->error, kErrOutOfBox);
      rec[s] = rr;
      fp += cell_fingerprint<D>(g, key, tab.ent[s].count);
      ++kc;
    }
  }
  if (lane == 0) {
    if (fp) atomicAdd((unsigned long long*)fp_out, (unsigned long long)fp);
    if (kc) atomicAdd(k_out, kc);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctrl->agg_done, 1u) == gridDim.x - 1) {
      ctrl->k[cur ^ 1] = 0;
      ctrl->agg_done = 0;
    }
  }
}

// Dense 3-D tables: tiled, separable 3x3x3 stencil.  A block owns an 8x8x8
// brick of lattice slots, stages the 10x10x10 halo of table entries in
// shared memory (SoA words, conflict-free) once, skips bricks with no
// occupied cell, and sums along z, then y, then x (3+3+3 adds instead of 27).
// Word sums are exact: the hi words are small signed integers and a low
// word's sum stays below 2^64 because a neighbourhood holds < 2^32 points.
// Occupied cells then round once and divide (grid.py:230-259,
// modeseek.py:109).  Also clears the previous table inside the brick and
// records k and the fingerprint.
// Bricks are 4 x 8 x 8 cells (x, y, z; z = the fastest key axis): 62.5 KB
// of shared memory and 256 threads, small enough to sit on an SM next to two
// k_shift_tma CTAs, so the side-stream table chain runs concurrently with
// the shift instead of in its tail.
constexpr int kBX = 4, kBY = 8, kBZ = 8;
constexpr int kHX = kBX + 2, kHY = kBY + 2, kHZ = kBZ + 2;
constexpr int kBrickCells = kBX * kBY * kBZ;        // 256
constexpr int kBrickThreads = kBrickCells;
constexpr int kMaskWords = kBrickCells / 32;        // occupancy bitmask words per brick
constexpr int kWords3 = 7;   // count, hi[3], lo[3]
constexpr int kH3 = kHX * kHY * kHZ;                // 600: staged halo / later the y-pass
constexpr int kS1 = kHX * kHY * kBZ;                // 480: z-pass
constexpr int kS2 = kHX * kBY * kBZ;                // 384: y-pass
constexpr size_t kBrickSmem = (size_t)(kH3 + kS1) * kWords3 * sizeof(u64) + kBrickCells * sizeof(u64);
constexpr int kSparseCells = 48;   // at most this many occupied cells: direct 27-point gathers

// Brick of a lattice slot (blockIdx order of the brick kernels).
struct BrickMap {
  u32 s0, s1, nby, nbz;
  __device__ __forceinline__ u32 of(u32 slot) const {
    const u32 x = slot / s0, r = slot - x * s0, y = r / s1, z = r - y * s1;
    return ((x / kBX) * nby + y / kBY) * nbz + z / kBZ;
  }
};

// First table of a sorted hash-table run, from the runs of the spatial sort:
// a run is one cell's points, contiguous in the sorted iterate, so a warp sums
// it (exact fixed point; 8 lanes per run) and writes its entry with plain stores after one
// insert -- no per-segment atomics (k_hist's hash path pays a CAS plus
// 2 d + 1 atomic adds per cell segment of a tile).
constexpr int kHistRunLanes = 8;   // lanes per run (a 4K RGB+xy image: ~14 points per run)

template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_hist_runs(const double* __restrict__ y, GridParams g, Tab tab,
                                                        const u32* __restrict__ runs, const u32* nruns,
                                                        const u32* __restrict__ start,
                                                        const u32* __restrict__ end, Ctrl* ctrl) {
  constexpr int G = kHistRunLanes;
  const u32 R = *nruns;
  const int sub = threadIdx.x & (G - 1);
  const i64 gg = ((i64)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const i64 ng = ((i64)gridDim.x * blockDim.x) / G;
  // (whole warps stay in the loop: the shuffles below are warp-wide)
  const i64 rounds = ((i64)R + ng - 1) / ng;
  for (i64 it = 0; it < rounds; ++it) {
    const i64 a = gg + it * ng;
    const bool live = a < (i64)R;
    const u32 r = live ? runs[a] : 0u;
    const u32 p0 = live ? start[r] : 0u, p1 = live ? end[r] : 0u;
    Agg<D> ag;
    ag.zero();
    for (u32 p = p0 + sub; p < p1; p += G) {
      ag.cnt += 1;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const i64 f = to_fixed(y[(i64)j * g.ld + p], g.qscale[j]);
        ag.hi[j] += f >> 32;
        ag.lo[j] += (u64)(f & 0xffffffffll);
      }
    }
#pragma unroll
    for (int off = G / 2; off; off >>= 1) {   // sum over the run's lane group
      ag.cnt += __shfl_xor_sync(kFull, ag.cnt, off);
#pragma unroll
      for (int j = 0; j < D; ++j) {
        ag.hi[j] += (i64)__shfl_xor_sync(kFull, (unsigned long long)ag.hi[j], off);
        ag.lo[j] += __shfl_xor_sync(kFull, ag.lo[j], off);
      }
    }
    if (sub == 0 && p1 > p0) {
      double v[D];
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = y[(i64)j * g.ld + p0];
      bool inside;
      const u64 key = pack_key<D>(g, v, inside);
      bool fresh;
      const u32 s = tab.insert(key, fresh, &ctrl->error);
      if (s != 0xffffffffu) {
        if (fresh) tab.list[atomicAdd(tab.k, 1u)] = s;
        Entry<D>* e = tab.ent + s;
        if (fresh) {               // (always: the runs are distinct cells)
          e->count = ag.cnt;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            e->hi[j] = (u64)ag.hi[j];
            e->lo[j] = ag.lo[j];
          }
        } else {
          atomicAdd(&e->count, (u64)ag.cnt);
#pragma unroll
          for (int j = 0; j < D; ++j) {
            atomicAdd(&e->hi[j], (u64)ag.hi[j]);
            atomicAdd(&e->lo[j], ag.lo[j]);
          }
        }
      }
    }
  }
}

// Brick occupancy of a freshly built table (the derived tables mark theirs
// in k_derive_brick3); occ zeroed before.
__global__ void __launch_bounds__(kThreads) k_mark_bricks(const Entry<3>* ent, u64 nslots, BrickMap bm, u8* occ) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x; s < (i64)nslots; s += stride)
    if (ent[s].count) occ[bm.of((u32)s)] = 1;
}

template <bool RS>
__global__ void __launch_bounds__(kBrickThreads) k_agg_brick3(GridParams g, DenseTable<3> tab, DenseTable<3> prev,
                                                              Rec<3>* __restrict__ rec, Ctrl* ctrl, u64* fp_out,
                                                              u32* k_out, int nbx, int nby, int nbz,
                                                              const u8* occ_cur, u8* occ_prev, const u32* pmask,
                                                              u32* cmask, int t, const double* __restrict__ rs) {
  if (block_stopped_before(ctrl, t)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* E = reinterpret_cast<u64*>(smem_raw);          // [7][kH3] halo, then [7][kS2] y-pass
  u64* S1 = E + (size_t)kWords3 * kH3;                // [7][kS1] z-pass
  u64* own = S1 + (size_t)kWords3 * kS1;              // [kBrickCells] own counts of the brick
  __shared__ int any;
  const i64 s0 = (i64)g.stride[0], s1 = (i64)g.stride[1];
  const int ext0 = (int)((i64)g.nkeys / s0), ext1 = (int)(s0 / s1), ext2 = (int)s1;
  const int bz = blockIdx.x % nbz, by = (blockIdx.x / nbz) % nby, bx = blockIdx.x / (nbz * nby);
  const int x0 = bx * kBX, y0 = by * kBY, z0 = bz * kBZ;
  const int tid = threadIdx.x;
  if (tid == 0) any = 0;
  const bool prev_occ = occ_prev[blockIdx.x] != 0, cur_occ = occ_cur[blockIdx.x] != 0;
  __syncthreads();
  if (prev_occ && tid == 0) occ_prev[blockIdx.x] = 0;
  // halo loads first (all of a thread's entries in flight at once; zeros
  // outside the lattice), then the previous table's clear, then the stores
  constexpr int HPT = (kH3 + kBrickThreads - 1) / kBrickThreads;
  Entry<3> v[HPT];
#pragma unroll
  for (int u = 0; u < HPT; ++u) {
    const int q = tid + u * kBrickThreads;
    v[u].count = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j) { v[u].hi[j] = 0; v[u].lo[j] = 0; }
    if (!cur_occ || q >= kH3) continue;
    const int hz = q % kHZ, hy = (q / kHZ) % kHY, hx = q / (kHZ * kHY);
    const int x = x0 + hx - 1, yv = y0 + hy - 1, z = z0 + hz - 1;
    if (x >= 0 && yv >= 0 && z >= 0 && x < ext0 && yv < ext1 && z < ext2) {
      const i64 sl = x * s0 + yv * s1 + z;
      if constexpr (RS) {
        // reference order: stage the count and the fp64 reference-order
        // sums (bit patterns in the hi words; the lo words stay unused)
        v[u].count = tab.ent[sl].count;
        if (v[u].count) {
#pragma unroll
          for (int j = 0; j < 3; ++j) v[u].hi[j] = __double_as_longlong(rs[sl * 3 + j]);
        }
      } else {
        v[u] = tab.ent[sl];
      }
    }
  }
  // clear the previous table in this brick (its cells are no longer read):
  // the occupancy bitmask its own k_agg_brick3 left (pmask) names the
  // entries, so nothing is read back
  {
    const u32 word = prev_occ ? pmask[(size_t)blockIdx.x * kMaskWords + (tid >> 5)] : 0u;
    if ((word >> (tid & 31)) & 1u) {
      const int z = z0 + tid % kBZ, yv = y0 + (tid / kBZ) % kBY, x = x0 + tid / (kBZ * kBY);
      Entry<3>* pe = prev.ent + (x * s0 + yv * s1 + z);
      pe->count = 0;
#pragma unroll
      for (int j = 0; j < 3; ++j) { pe->hi[j] = 0; pe->lo[j] = 0; }
    }
  }
  if (!cur_occ) {
    if ((tid & 31) == 0) cmask[(size_t)blockIdx.x * kMaskWords + (tid >> 5)] = 0u;
    return;
  }
  int occ = 0;
#pragma unroll
  for (int u = 0; u < HPT; ++u) {
    const int q = tid + u * kBrickThreads;
    if (q >= kH3) continue;
    const int hz = q % kHZ, hy = (q / kHZ) % kHY, hx = q / (kHZ * kHY);
    E[0 * kH3 + q] = v[u].count;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      E[(1 + j) * kH3 + q] = v[u].hi[j];
      E[(4 + j) * kH3 + q] = v[u].lo[j];
    }
    if (hx >= 1 && hx <= kBX && hy >= 1 && hy <= kBY && hz >= 1 && hz <= kBZ) {
      own[((hx - 1) * kBY + (hy - 1)) * kBZ + (hz - 1)] = v[u].count;
      occ |= v[u].count != 0;
    }
  }
  if (occ) any = 1;
  __shared__ int nocc;
  if (tid == 0) nocc = 0;
  __syncthreads();
  {
    const unsigned bits = __ballot_sync(kFull, own[tid] != 0);   // one thread per brick cell
    if ((tid & 31) == 0) {
      cmask[(size_t)blockIdx.x * kMaskWords + (tid >> 5)] = bits;
      if (bits) atomicAdd(&nocc, __popc(bits));
    }
  }
  if (!any) return;
  __syncthreads();
  // sparse brick (few occupied cells, typical once clusters contract): each
  // occupied cell gathers its 27 neighbours from the staged halo directly;
  // dense brick: separable z, y, x passes over the whole brick
  const bool sparse = RS || nocc <= kSparseCells;
  if (!sparse) {
    // z-pass: S1[hx][hy][z] = E[hx][hy][z] + E[hx][hy][z+1] + E[hx][hy][z+2]
    for (int q = tid; q < kS1; q += blockDim.x) {
      const int z = q % kBZ, hy = (q / kBZ) % kHY, hx = q / (kBZ * kHY);
      const int b0 = (hx * kHY + hy) * kHZ + z;
#pragma unroll
      for (int w = 0; w < kWords3; ++w)
        S1[w * kS1 + q] = E[w * kH3 + b0] + E[w * kH3 + b0 + 1] + E[w * kH3 + b0 + 2];
    }
    __syncthreads();
    // y-pass into E: S2[hx][y][z] = S1[hx][y][z] + S1[hx][y+1][z] + S1[hx][y+2][z]
    for (int q = tid; q < kS2; q += blockDim.x) {
      const int z = q % kBZ, yv = (q / kBZ) % kBY, hx = q / (kBZ * kBY);
      const int b0 = (hx * kHY + yv) * kBZ + z;
#pragma unroll
      for (int w = 0; w < kWords3; ++w)
        E[w * kS2 + q] = S1[w * kS1 + b0] + S1[w * kS1 + b0 + kBZ] + S1[w * kS1 + b0 + 2 * kBZ];
    }
    __syncthreads();
  }
  // x-pass (or direct gather) + targets for the occupied cells
  u64 fp = 0;
  u32 kc = 0;
  for (int q = tid; q < kBrickCells; q += blockDim.x) {
    const u64 mine = own[q];
    if (mine == 0) continue;
    const int lz = q % kBZ, ly = (q / kBZ) % kBY, lx = q / (kBZ * kBY);
    u64 wsum[kWords3];
    if constexpr (RS) {
      // 27 neighbours in lexicographic offset order (dx, dy, dz; grid.py:
      // 199-208), each present one added in fp64 (grid.py:253-258)
      u64 cn = 0;
      double sm[3] = {0.0, 0.0, 0.0};
      for (int dx = 0; dx < 3; ++dx)
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dz = 0; dz < 3; ++dz) {
            const int h0 = ((lx + dx) * kHY + (ly + dy)) * kHZ + lz + dz;
            const u64 cc = E[h0];
            if (cc) {
              cn += cc;
#pragma unroll
              for (int j = 0; j < 3; ++j) sm[j] = __dadd_rn(sm[j], __longlong_as_double((long long)E[(1 + j) * kH3 + h0]));
            }
          }
      const u64 slot = (u64)(x0 + lx) * s0 + (u64)(y0 + ly) * s1 + (u64)(z0 + lz);
      Rec<3> r;
      const double c = (double)cn;
#pragma unroll
      for (int j = 0; j < 3; ++j) r.t[j] = __ddiv_rn(sm[j], c);
      bool inside;
      r.key = pack_key<3>(g, r.t, inside);
      if (!inside) atomicOr(&ctrl->error, kErrOutOfBox);
      rec[slot] = r;
      fp += cell_fingerprint<3>(g, slot, mine);
      ++kc;
      continue;
    }
    if (sparse) {
#pragma unroll
      for (int w = 0; w < kWords3; ++w) wsum[w] = 0;
      for (int dx = 0; dx < 3; ++dx)
        for (int dy = 0; dy < 3; ++dy) {
          const int h0 = ((lx + dx) * kHY + (ly + dy)) * kHZ + lz;
#pragma unroll
          for (int w = 0; w < kWords3; ++w)
            wsum[w] += E[w * kH3 + h0] + E[w * kH3 + h0 + 1] + E[w * kH3 + h0 + 2];
        }
    } else {
      const int b0 = (lx * kBY + ly) * kBZ + lz;
#pragma unroll
      for (int w = 0; w < kWords3; ++w)
        wsum[w] = E[w * kS2 + b0] + E[w * kS2 + b0 + kBY * kBZ] + E[w * kS2 + b0 + 2 * kBY * kBZ];
    }
    const u64 slot = (u64)(x0 + lx) * s0 + (u64)(y0 + ly) * s1 + (u64)(z0 + lz);
    Rec<3> r;
    const double c = (double)wsum[0];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const i128 v = (((i128)(i64)wsum[1 + j]) << 32) + (i128)wsum[4 + j];
      r.t[j] = __ddiv_rn(i128_to_double(v, -g.qexp[j]), c);
    }
    bool inside;
    r.key = pack_key<3>(g, r.t, inside);
    if (!inside) atomicOr(&ctrl->error, kErrOutOfBox);
    rec[slot] = r;
    fp += cell_fingerprint<3>(g, slot, mine);
    ++kc;
  }
  for (int o = 16; o; o >>= 1) {
    fp += __shfl_xor_sync(kFull, fp, o);
    kc += __shfl_xor_sync(kFull, kc, o);
  }
  if ((tid & 31) == 0) {
    if (fp) atomicAdd((unsigned long long*)fp_out, (unsigned long long)fp);
    if (kc) atomicAdd(k_out, kc);
  }
}

// Table of y_{t+1} from the table of y_t.  Every point of occupied cell c
// moves to exactly target_c (modeseek.py:109: y' depends on the cell only),
// so the per-point histogram of y_{t+1} (grid.py:179-190) equals
//     count[key(target_c)] += count_c,  sums[key(target_c)] += count_c * fixed(target_c)
// summed over c -- an identity over integers, hence bit-identical to binning
// the points (tests: per-iteration fingerprints and the exact model).
// Dense tables are walked in key order (adjacent cells tend to share a
// target cell); the buffer receiving the new table was cleared by k_agg.
template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_derive(GridParams g, Tab cur, Tab nxt, const Rec<D>* __restrict__ rec,
                                                     Ctrl* ctrl, int c, int t, u32* nsrc = nullptr) {
  if (block_stopped_before(ctrl, t)) return;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const i64 items = Tab::kDense ? (i64)g.nkeys : (i64)ctrl->k[c];
  for (i64 a = tid; a < items; a += stride) {
    const u32 s = Tab::kDense ? (u32)a : cur.list[a];
    const u64 cnt = cur.ent[s].count;
    if (cnt == 0) continue;
    const Rec<D> r = rec[s];
    Agg<D> ag;
    ag.cnt = (u32)cnt;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const i64 f = to_fixed(r.t[j], g.qscale[j]);
      ag.hi[j] = (f >> 32) * (i64)cnt;
      ag.lo[j] = (u64)(f & 0xffffffffll) * cnt;
    }
    flush_segment<D, Tab, false>(nxt, ctrl, r.key, ag);
    // reference-order sums: how many source cells reach the target
    if (nsrc) atomicAdd(nsrc + nxt.lookup(r.key), 1u);
  }
}

// k_derive for dense 3-D tables, one block per occupied brick; marks the
// bricks of the new table (occ_nxt was reset by k_agg_brick3).
__global__ void __launch_bounds__(kBrickThreads) k_derive_brick3(GridParams g, DenseTable<3> cur, DenseTable<3> nxt,
                                                                 const Rec<3>* __restrict__ rec, Ctrl* ctrl,
                                                                 int nby, int nbz, BrickMap bm, const u8* occ_cur,
                                                                 u8* occ_nxt, const u32* cmask, int t,
                                                                 u32* nsrc) {
  if (block_stopped_before(ctrl, t)) return;
  if (!occ_cur[blockIdx.x]) return;
  // the brick's cell-occupancy mask (written by k_agg_brick3 for this table)
  // spares the count reads of empty cells
  const bool mine = (cmask[(size_t)blockIdx.x * kMaskWords + (threadIdx.x >> 5)] >> (threadIdx.x & 31)) & 1u;
  const i64 s0 = (i64)g.stride[0], s1 = (i64)g.stride[1];
  const int ext0 = (int)((i64)g.nkeys / s0), ext1 = (int)(s0 / s1), ext2 = (int)s1;
  const int bz = blockIdx.x % nbz, by = (blockIdx.x / nbz) % nby, bx = blockIdx.x / (nbz * nby);
  const int q = threadIdx.x;
  const int z = bz * kBZ + q % kBZ, yv = by * kBY + (q / kBZ) % kBY, x = bx * kBX + q / (kBZ * kBY);
  const bool inside = x < ext0 && yv < ext1 && z < ext2;
  const u32 s = inside ? (u32)(x * s0 + yv * s1 + z) : 0u;
  const u64 cnt = (inside && mine) ? cur.ent[s].count : 0;
  u64 key = kEmpty;
  Agg<3> ag;
  ag.zero();
  if (cnt) {
    const Rec<3> r = rec[s];
    key = r.key;
    ag.cnt = (u32)cnt;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const i64 f = to_fixed(r.t[j], g.qscale[j]);
      ag.hi[j] = (f >> 32) * (i64)cnt;
      ag.lo[j] = (u64)(f & 0xffffffffll) * cnt;
    }
  }
  // cells of a warp moving to one target cell (common once clusters
  // contract) flush once: exact integer sums over the peers
  if (__all_sync(kFull, key == kEmpty)) return;
  const unsigned peers = __match_any_sync(kFull, key);
  const int lane = threadIdx.x & 31;
  if (__any_sync(kFull, __popc(peers) > 1)) {
    // reduce each peer group to its lowest lane: in round k the lane of
    // group rank r adds the partial of rank r + 2^k (pointer doubling)
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const unsigned src = __fns(peers, lane, (1 << k) + 1);
      const int from = src < 32 ? (int)src : lane;
      const u32 oc = __shfl_sync(kFull, ag.cnt, from);
      i64 oh[3];
      u64 ol[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        oh[j] = __shfl_sync(kFull, ag.hi[j], from);
        ol[j] = __shfl_sync(kFull, ag.lo[j], from);
      }
      if (src < 32) {
        ag.cnt += oc;
#pragma unroll
        for (int j = 0; j < 3; ++j) { ag.hi[j] += oh[j]; ag.lo[j] += ol[j]; }
      }
    }
  }
  if (key == kEmpty || lane != __ffs(peers) - 1) return;
  flush_segment<3, DenseTable<3>, false>(nxt, ctrl, key, ag);
  if (nsrc) atomicAdd(nsrc + key, (u32)__popc(peers));   // source cells reaching the target
  if (key < g.nkeys) occ_nxt[bm.of((u32)key)] = 1;
}

// Dense tables: occupied-cell list from the counts (warp-aggregated append).
template <int D>
__global__ void __launch_bounds__(kThreads) k_compact(const Entry<D>* ent, u64 nslots, u32* list, u32* kp) {
  const int lane = threadIdx.x & 31;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const i64 t0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  for (i64 base = t0 - lane; base < (i64)nslots; base += stride) {
    const i64 s = base + lane;
    const bool occ = s < (i64)nslots && ent[s].count != 0;
    const u32 m = __ballot_sync(kFull, occ);
    u32 at = 0;
    if (lane == 0 && m) at = atomicAdd(kp, (u32)__popc(m));
    at = __shfl_sync(kFull, at, 0);
    if (occ) list[at + __popc(m & ((1u << lane) - 1u))] = (u32)s;
  }
}

// Dense tables: zero every occupied slot (no list needed).
template <int D>
__global__ void __launch_bounds__(kThreads) k_clear_all(Entry<D>* ent, u64 nslots) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 s = (i64)blockIdx.x * blockDim.x + threadIdx.x; s < (i64)nslots; s += stride) {
    Entry<D>* e = ent + s;
    if (e->count) {
      e->count = 0;
#pragma unroll
      for (int j = 0; j < D; ++j) { e->hi[j] = 0; e->lo[j] = 0; }
    }
  }
}

// ---------------------------------------------------------------- k_agg

template <int D, class Tab>
__device__ __forceinline__ void neighbourhood_sum(const GridParams& g, const Tab& tab, u64 key,
                                                  u64& cnt, i128* sum) {
  constexpr int M = (D == 1) ? 3 : (D == 2) ? 9 : (D == 3) ? 27 : (D == 4) ? 81 :
                    (D == 5) ? 243 : (D == 6) ? 729 : (D == 7) ? 2187 : 6561;
  cnt = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) sum[j] = 0;
  for (int o = 0; o < M; ++o) {
    int r = o;
    i64 delta = 0;
#pragma unroll
    for (int j = D - 1; j >= 0; --j) {
      delta += (i64)((r % 3) - 1) * (i64)g.stride[j];
      r /= 3;
    }
    u32 ns;
    if (tab.find(key + (u64)delta, ns)) {
      const Entry<D>& e = tab.ent[ns];
      cnt += e.count;
#pragma unroll
      for (int j = 0; j < D; ++j) sum[j] += (((i128)(i64)e.hi[j]) << 32) + (i128)e.lo[j];
    }
  }
}

// ------------------------------------------------------- neighbourhood sums
// grid.py:253-258: hits in lexicographic offset order, each added in fp64
// to an accumulator starting at 0.0; counts exact.

template <int D, class Tab>
__device__ __forceinline__ void neighbourhood_sum_rs(const GridParams& g, const Tab& tab, const double* __restrict__ rs,
                                                     u64 key, u64& cnt, double* sum) {
  constexpr int M = (D == 1) ? 3 : (D == 2) ? 9 : (D == 3) ? 27 : (D == 4) ? 81 :
                    (D == 5) ? 243 : (D == 6) ? 729 : (D == 7) ? 2187 : 6561;
  cnt = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) sum[j] = 0.0;
  for (int o = 0; o < M; ++o) {
    int r = o;
    i64 delta = 0;
#pragma unroll
    for (int j = D - 1; j >= 0; --j) {
      delta += (i64)((r % 3) - 1) * (i64)g.stride[j];
      r /= 3;
    }
    u32 ns;
    if (tab.find(key + (u64)delta, ns)) {
      cnt += tab.ent[ns].count;
#pragma unroll
      for (int j = 0; j < D; ++j) sum[j] = __dadd_rn(sum[j], rs[(i64)ns * D + j]);
    }
  }
}

template <int D, class Tab>
__device__ __forceinline__ void agg_cell(const GridParams& g, const Tab& tab, u32 s, Rec<D>* __restrict__ rec,
                                         u64& fp, Ctrl* ctrl, const double* __restrict__ rs) {
  const u64 key = tab.key_of(s);
  u64 cnt;
  Rec<D> r;
  if (rs) {
    // reference order (grid.py:253-258, modeseek.py:109)
    double sum[D];
    neighbourhood_sum_rs<D>(g, tab, rs, key, cnt, sum);
    const double c = (double)cnt;
#pragma unroll
    for (int j = 0; j < D; ++j) r.t[j] = __ddiv_rn(sum[j], c);
  } else {
    i128 sum[D];
    neighbourhood_sum<D>(g, tab, key, cnt, sum);
    const double c = (double)cnt;
#pragma unroll
    for (int j = 0; j < D; ++j) r.t[j] = __ddiv_rn(i128_to_double(sum[j], -g.qexp[j]), c);
  }
  bool inside;
  r.key = pack_key<D>(g, r.t, inside);
  if (!inside) atomicOr(&ctrl->error, kErrOutOfBox);
  rec[s] = r;
  fp += cell_fingerprint<D>(g, key, tab.ent[s].count);
}

// Per occupied cell: 3^d neighbourhood -> target record.  Dense tables are
// walked slot by slot (empty slots are one 8-byte read); hash tables by
// their occupied list.  Also clears the previous iteration's table (the
// next k_derive fills it) and records k and the (cells, counts) fingerprint
// of this iteration; the last CTA resets the cleared table's cell count.
template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_agg(GridParams g, Tab tab, Tab prev, Rec<D>* __restrict__ rec,
                                                  Ctrl* ctrl, int cur, u64* fp_out, u32* k_out, int t,
                                                  const double* __restrict__ rs = nullptr) {
  if (block_stopped_before(ctrl, t)) return;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const i64 tid = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 fp = 0;
  u32 kc = 0;
  if constexpr (Tab::kDense) {
    const i64 ns = (i64)g.nkeys;
    for (i64 s = tid; s < ns; s += stride) {
      Entry<D>* e = prev.ent + s;
      if (e->count) {
        e->count = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) { e->hi[j] = 0; e->lo[j] = 0; }
      }
    }
    for (i64 s = tid; s < ns; s += stride) {
      if (tab.ent[s].count == 0) continue;
      agg_cell<D>(g, tab, (u32)s, rec, fp, ctrl, rs);
      ++kc;
    }
  } else {
    const u32 kp = ctrl->k[cur ^ 1];
    for (i64 a = tid; a < kp; a += stride) {
      const u32 s = prev.list[a];
      Entry<D>* e = prev.ent + s;
      e->count = 0;
#pragma unroll
      for (int j = 0; j < D; ++j) { e->hi[j] = 0; e->lo[j] = 0; }
      prev.keys[s] = kEmpty;
    }
    const u32 k = ctrl->k[cur];
    for (i64 a = tid; a < k; a += stride) {
      agg_cell<D>(g, tab, tab.list[a], rec, fp, ctrl, rs);
      ++kc;
    }
  }
  for (int o = 16; o; o >>= 1) {
    fp += __shfl_xor_sync(kFull, fp, o);
    kc += __shfl_xor_sync(kFull, kc, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (fp) atomicAdd((unsigned long long*)fp_out, (unsigned long long)fp);
    if (kc) atomicAdd(k_out, kc);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctrl->agg_done, 1u) == gridDim.x - 1) {
      ctrl->k[cur ^ 1] = 0;   // every CTA has read it: the next k_derive appends from 0
      ctrl->agg_done = 0;
    }
  }
}

// ------------------------------------------------------------ spatial sort
// One-time counting sort of the points by their initial cell (count-only
// k_hist -> exclusive scan of the occupied cells' counts -> scatter).  All
// later reductions are exact integer sums, so the order inside a cell is
// irrelevant to the results; what the sort buys is that every warp sees
// runs of equal cells -- and, from iteration 1 on, runs of identical
// positions -- so the table atomics collapse to one per run.

constexpr int kScanItems = 8;
constexpr int kScanChunk = kThreads * kScanItems;

template <int D>
__device__ __forceinline__ u64 entry_count(const Entry<D>* ent, u32 s) { return ent[s].count; }

// Items are either the entries of an occupied list (list != nullptr, count
// *kp) or, for dense tables, every slot in key order (count nslots) -- the
// latter makes the sorted point order the lexicographic cell order.
__device__ __forceinline__ u32 scan_item(const u32* list, i64 a) { return list ? list[a] : (u32)a; }
// counts come from the table entries, or from a plain u32 array (cnt32)
template <int D>
__device__ __forceinline__ u64 item_count(const Entry<D>* ent, const u32* cnt32, u32 s) {
  return cnt32 ? (u64)cnt32[s] : ent[s].count;
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_scan_reduce(const Entry<D>* ent, const u32* list, const u32* kp,
                                                          u64* bsum, u64 nslots, const u32* cnt32 = nullptr) {
  const u64 k = list ? (u64)*kp : nslots;
  const i64 a0 = (i64)blockIdx.x * kScanChunk;
  u64 s = 0;
  if (a0 < k) {
    for (int it = 0; it < kScanItems; ++it) {
      const i64 a = a0 + (i64)it * kThreads + threadIdx.x;
      if (a < (i64)k) s += item_count<D>(ent, cnt32, scan_item(list, a));
    }
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  __shared__ u64 w[kThreads / 32];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 t = 0;
    for (int q = 0; q < kThreads / 32; ++q) t += w[q];
    bsum[blockIdx.x] = t;
  }
}

// exclusive scan of nb block sums, single block
__global__ void __launch_bounds__(1024) k_scan_top(u64* bsum, int nb) {
  __shared__ u64 w[32];
  __shared__ u64 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const u64 v = i < nb ? bsum[i] : 0;
    u64 x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const u64 y = __shfl_up_sync(kFull, x, o);
      if ((threadIdx.x & 31) >= o) x += y;
    }
    if ((threadIdx.x & 31) == 31) w[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      u64 z = w[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const u64 y = __shfl_up_sync(kFull, z, o);
        if (threadIdx.x >= o) z += y;
      }
      w[threadIdx.x] = z;
    }
    __syncthreads();
    const u64 before = (threadIdx.x >= 32 ? w[(threadIdx.x >> 5) - 1] : 0) + x - v;
    if (i < nb) bsum[i] = carry + before;
    __syncthreads();
    if (threadIdx.x == 1023) carry += before + v;
    __syncthreads();
  }
}

// per-cell write cursor = exclusive prefix of counts (list order)
template <int D>
__global__ void __launch_bounds__(kThreads) k_scan_apply(const Entry<D>* ent, const u32* list, const u32* kp,
                                                         const u64* bsum, u32* off, u64 nslots, u32* start,
                                                         const u32* cnt32 = nullptr) {
  const u64 k = list ? (u64)*kp : nslots;
  const i64 a0 = (i64)blockIdx.x * kScanChunk;
  if (a0 >= (i64)k) return;
  // thread t owns items a0 + t*kScanItems .. +kScanItems-1 (contiguous)
  u64 c[kScanItems];
  u64 tot = 0;
  for (int it = 0; it < kScanItems; ++it) {
    const i64 a = a0 + (i64)threadIdx.x * kScanItems + it;
    c[it] = a < (i64)k ? item_count<D>(ent, cnt32, scan_item(list, a)) : 0;
    tot += c[it];
  }
  u64 x = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const u64 y = __shfl_up_sync(kFull, x, o);
    if ((threadIdx.x & 31) >= o) x += y;
  }
  __shared__ u64 w[kThreads / 32];
  if ((threadIdx.x & 31) == 31) w[threadIdx.x >> 5] = x;
  __syncthreads();
  u64 pre = bsum[blockIdx.x] + x - tot;
  for (int q = 0; q < (int)(threadIdx.x >> 5); ++q) pre += w[q];
  for (int it = 0; it < kScanItems; ++it) {
    const i64 a = a0 + (i64)threadIdx.x * kScanItems + it;
    if (a < (i64)k) {
      off[scan_item(list, a)] = (u32)pre;
      if (start) start[scan_item(list, a)] = (u32)pre;
    }
    pre += c[it];
  }
}

// scatter points into cell order; warp-aggregated cursor bumps.  Also
// records, for the run-based extraction, each point's initial cell slot in
// ORIGINAL order (coalesced) and each run's minimum original index.
// Scatter target: whole AoS records (D doubles padded to 16-byte multiples),
// so every random write covers full 32-byte sectors (no partial-sector
// read-modify-write); k_unstage transposes back to SoA with coalesced I/O.
template <int D>
struct StageRec {
  static constexpr int W = (D + 1) & ~1;   // doubles per record
};

template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_scatter(const double* __restrict__ y, double* __restrict__ stage, i64 n,
                                                      GridParams g, Tab tab, u32* off, u32* perm, u32* cell0,
                                                      u32* minidx, Ctrl* ctrl) {
  const int lane = threadIdx.x & 31;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 base = warp * 32; base < n; base += nwarps * 32) {
    const i64 i = base + lane;
    double v[D];
    u32 s = 0xffffffffu;
    if (i < n) {
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = __ldcs(y + (i64)j * g.ld + i);
      bool inside;
      const u64 key = pack_key<D>(g, v, inside);
      if (!inside || !tab.find(key, s)) { atomicOr(&ctrl->error, kErrMissing); s = 0xffffffffu; }
      cell0[i] = s;
    }
    const unsigned peers = __match_any_sync(kFull, s);
    const int leader = __ffs(peers) - 1;
    const u32 mi = __reduce_min_sync(peers, (u32)i);
    u32 basepos = 0;
    if (lane == leader && s != 0xffffffffu) {
      basepos = atomicAdd(off + s, (u32)__popc(peers));
      atomicMin(minidx + s, mi);
    }
    basepos = __shfl_sync(kFull, basepos, leader);
    if (s != 0xffffffffu) {
      const u32 pos = basepos + __popc(peers & ((1u << lane) - 1u));
      constexpr int W = StageRec<D>::W;
      double2* dst = reinterpret_cast<double2*>(stage + (i64)pos * W);
#pragma unroll
      for (int q = 0; q < W / 2; ++q)
        dst[q] = make_double2(v[2 * q], (2 * q + 1 < D) ? v[2 * q + 1] : 0.0);
      if (perm) perm[pos] = (u32)i;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads) k_unstage(const double* __restrict__ stage, double* __restrict__ ys, i64 n,
                                                      i64 ld) {
  constexpr int W = StageRec<D>::W;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double2* src = reinterpret_cast<const double2*>(stage + i * W);
    double v[W];
#pragma unroll
    for (int q = 0; q < W / 2; ++q) {
      const double2 a = __ldcs(src + q);
      v[2 * q] = a.x;
      v[2 * q + 1] = a.y;
    }
#pragma unroll
    for (int j = 0; j < D; ++j) __stcs(ys + (i64)j * ld + i, v[j]);
  }
}

// Run-based extraction (after the spatial sort, at least one iteration).
// A run = the points of one initial cell: contiguous in sorted order and,
// from iteration 1 on, bitwise-identical positions.  Per run: its final
// cell's component root (stored over the run's cursor slot) and the
// first-appearance minimum over its original indices (modeseek.py:262-265).
template <int D, class Tab>
__global__ void k_run_first(const double* __restrict__ yf, GridParams g, Tab tab, const u32* runs,
                            const u32* nruns, const u32* start, const u32* minidx, const u32* par,
                            u32* first, u32* runroot, Ctrl* ctrl, u32 offset, const double* runpos, i64 rld) {
  const u32 R = *nruns;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < R; a += stride) {
    const u32 s0 = runs[a];
    double v[D];
    if (runpos) {
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = runpos[(i64)j * rld + a];
    } else {
      const u32 p = start[s0];
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = yf[(i64)j * g.ld + p];
    }
    bool inside;
    const u64 key = pack_key<D>(g, v, inside);
    u32 sf = 0;
    if (!inside || !tab.find(key, sf)) { atomicOr(&ctrl->error, kErrMissing); continue; }
    const u32 r = par[sf];
    runroot[s0] = r;
    atomicMin(first + r, minidx[s0] + offset);
  }
}

// per-cell labels of the initial cells (host delivery: the host expands
// them through its copy of cell0; k_labels_runs's values)
__global__ void __launch_bounds__(kThreads) k_slot_labels(const u32* __restrict__ runs, const u32* nruns,
                                                          const u32* __restrict__ runroot,
                                                          const u32* __restrict__ rankmap, u32* slotlab) {
  const u32 R = *nruns;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < R; a += stride) {
    const u32 s0 = runs[a];
    slotlab[s0] = rankmap[runroot[s0]];
  }
}

// Per-segment colour sums and pixel counts of a segmentation
// (segment_map_from_labeling, segment.py:109-117): pixel i carries label
// slotlab[cell0[i]] (host label delivery) or labels[i].  uint8 colours sum
// exactly in integers, so the means (sum / count in fp64) equal np.bincount's.
// Lanes of a warp with the same label combine before the atomics
// (neighbouring pixels mostly share a segment).  out: [label][4] = r, g, b, n.
__global__ void __launch_bounds__(kThreads) k_label_colors(const unsigned char* __restrict__ pix, i64 n,
                                                           const u32* __restrict__ cell0,
                                                           const u32* __restrict__ slotlab,
                                                           const i64* __restrict__ labels, u64* out) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (i64 i0 = (i64)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
    const i64 i = i0 + lane;
    u32 lab = 0xffffffffu, r = 0, g = 0, b = 0;
    if (i < n) {
      lab = cell0 ? slotlab[cell0[i]] : (u32)labels[i];
      r = pix[i * 3];
      g = pix[i * 3 + 1];
      b = pix[i * 3 + 2];
    }
    const unsigned peers = __match_any_sync(kFull, lab);
    const u32 sr = __reduce_add_sync(peers, r), sg = __reduce_add_sync(peers, g), sb = __reduce_add_sync(peers, b);
    if (lab != 0xffffffffu && lane == __ffs(peers) - 1) {
      u64* o = out + (i64)lab * 4;
      atomicAdd(reinterpret_cast<unsigned long long*>(o), (unsigned long long)sr);
      atomicAdd(reinterpret_cast<unsigned long long*>(o + 1), (unsigned long long)sg);
      atomicAdd(reinterpret_cast<unsigned long long*>(o + 2), (unsigned long long)sb);
      atomicAdd(reinterpret_cast<unsigned long long*>(o + 3), (unsigned long long)__popc(peers));
    }
  }
}

// labels of the first n points from the per-cell labels (host delivery: this
// part is copied to a pinned caller buffer while host threads expand the rest)
__global__ void __launch_bounds__(kThreads) k_labels_from_slots(const u32* __restrict__ cell0, i64 n,
                                                                const u32* __restrict__ slotlab, i64* labels) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 c = cell0[i];
    labels[i] = c == 0xffffffffu ? -1 : (i64)slotlab[c];
  }
}

// labels in original order: one coalesced pass (cell0 -> run root -> rank)
__global__ void __launch_bounds__(kThreads) k_labels_runs(const u32* __restrict__ cell0, i64 n,
                                                          const u32* __restrict__ runroot,
                                                          const u32* __restrict__ rankmap, i64* labels) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 s0 = cell0[i];   // 0xffffffff only after a flagged lookup failure
    labels[i] = s0 == 0xffffffffu ? -1 : (i64)rankmap[runroot[s0]];
  }
}

// ------------------------------------------- two-level sort (dense tables)
// The one-time spatial sort without per-point global atomics:
//   k_bk_count   per block chunk: shared-memory histogram of coarse buckets
//                (2^shift consecutive slots), each point's slot -> cell0
//   k_bk_cols    per bucket: exclusive scan over the blocks (in place)
//   k_bk_stage   per block chunk, in rounds of kStageRound points: local
//                counting sort by bucket in shared memory, then coalesced
//                writes of bucket runs into the bucket-grouped staging buffer
//   k_bk_tally   per fixed-size chunk of staging (load-balanced whatever the
//                bucket sizes): shared-memory count / min index per slot,
//                one global atomic pair per (chunk, slot) -> run sizes + minima
//   (scan of the run sizes over slots -> run starts / cursors)
//   k_bk_place   per chunk again: per-slot cursor bump once per (chunk, slot),
//                shared-memory local ranks, SoA fp64 writes of the sorted iterate
// The passes read the INPUT rows directly (SrcAoS: fp32/fp64 (n, d) as the
// caller passed them, upcast exactly like PointSet, grid.py:43) or the fp64
// iterate (SrcSoA, image features).  Staging records carry the source-type
// coordinates and the original index only (16 B for fp32 d=3); the slot is
// recomputed from the coordinates where needed (bitwise the same key).
// Chunks whose slots span more than the shared-memory window fall back to
// per-record global atomics (correct, just slower; never seen on the configs).
template <int D, typename T>
struct SrcAoS {
  using RT = T;
  const T* x;
  __device__ __forceinline__ void raw(i64 i, RT (&r)[D]) const {
#pragma unroll
    for (int j = 0; j < D; ++j) r[j] = __ldcs(x + i * D + j);
  }
};

template <int D>
struct SrcSoA {
  using RT = double;
  const double* y;
  i64 ld;
  __device__ __forceinline__ void raw(i64 i, RT (&r)[D]) const {
#pragma unroll
    for (int j = 0; j < D; ++j) r[j] = __ldcs(y + (i64)j * ld + i);
  }
};

// Staging record: D coordinates of type RT, then the original index; padded
// to whole 16-byte vectors.
template <int D, typename RT>
struct SRec {
  static constexpr int kBytes = ((int)(D * sizeof(RT)) + 4 + 15) & ~15;
  static constexpr int kVec = kBytes / 16;    // uint4 per record
  static constexpr int kIdxWord = (int)(D * sizeof(RT)) / 4;
};

template <int D, typename RT>
__device__ __forceinline__ void srec_put(u32* w, const RT (&r)[D], u32 idx) {
  RT* c = reinterpret_cast<RT*>(w);
#pragma unroll
  for (int j = 0; j < D; ++j) c[j] = r[j];
  w[SRec<D, RT>::kIdxWord] = idx;
#pragma unroll
  for (int k = SRec<D, RT>::kIdxWord + 1; k < SRec<D, RT>::kBytes / 4; ++k) w[k] = 0u;
}

// slot of a staged record (the upcast is exact, so this is the key k_bk_count saw)
template <int D, typename RT>
__device__ __forceinline__ u32 srec_slot(const GridParams& g, const uint4* rec, double (&v)[D], u32& idx,
                                         bool& inside) {
  u32 w[SRec<D, RT>::kBytes / 4];
#pragma unroll
  for (int k = 0; k < SRec<D, RT>::kVec; ++k) {
    const uint4 q = rec[k];
    w[4 * k] = q.x; w[4 * k + 1] = q.y; w[4 * k + 2] = q.z; w[4 * k + 3] = q.w;
  }
  const RT* c = reinterpret_cast<const RT*>(w);
#pragma unroll
  for (int j = 0; j < D; ++j) v[j] = (double)c[j];
  idx = w[SRec<D, RT>::kIdxWord];
  return (u32)pack_key<D>(g, v, inside);
}

// coordinates of a staged record, upcast
template <int D, typename RT>
__device__ __forceinline__ void srec_coords(const uint4* rec, double (&v)[D]) {
  u32 w[SRec<D, RT>::kBytes / 4];
#pragma unroll
  for (int k = 0; k < SRec<D, RT>::kVec; ++k) {
    const uint4 q = rec[k];
    w[4 * k] = q.x; w[4 * k + 1] = q.y; w[4 * k + 2] = q.z; w[4 * k + 3] = q.w;
  }
  const RT* c = reinterpret_cast<const RT*>(w);
#pragma unroll
  for (int j = 0; j < D; ++j) v[j] = (double)c[j];
}

constexpr int kChunkRecs = 4096;   // k_bk_tally chunk (k_bk_place uses half)
constexpr int kBucketShiftMin = 12;        // >= 4096 slots per coarse bucket
constexpr int kTallyWin = 2 << kBucketShiftMin;   // a chunk spans <= 2 buckets when they are full

// Shared-memory counter bump returning each lane's rank.  __match_any_sync
// saturates the ADU pipe at one match per point, so: one atomic for a warp
// whose lanes all hit the same counter (sorted inputs, hot cells), plain
// per-lane shared atomics otherwise (random inputs rarely collide).
__device__ __forceinline__ u32 smem_bump(u32* ctr, u32 key, bool valid) {
  const int lane = threadIdx.x & 31;
  const u32 k0 = __shfl_sync(kFull, key, 0);
  if (__all_sync(kFull, valid && key == k0)) {
    u32 b = 0;
    if (lane == 0) b = atomicAdd(ctr + k0, 32u);
    return __shfl_sync(kFull, b, 0) + lane;
  }
  return valid ? atomicAdd(ctr + key, 1u) : 0u;
}

template <int D, class Src>
__global__ void __launch_bounds__(kThreads) k_bk_count(Src src, i64 n, GridParams g, int shift, u32 nb, i64 chunk,
                                                       u32* blk_counts, u32* cell0, Ctrl* ctrl) {
  using RT = typename Src::RT;
  extern __shared__ u32 hist[];
  for (u32 b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const i64 a0 = (i64)blockIdx.x * chunk, a1 = min(n, a0 + chunk);
  for (i64 base = a0; base < a1; base += blockDim.x) {
    const i64 i = base + threadIdx.x;
    u32 bk = 0xffffffffu;
    if (i < a1) {
      RT r[D];
      src.raw(i, r);
      double v[D];
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = (double)r[j];
      bool inside;
      const u64 key = pack_key<D>(g, v, inside);
      if (!inside) {
        atomicOr(&ctrl->error, kErrMissing);
        cell0[i] = 0xffffffffu;
      } else {
        cell0[i] = (u32)key;
        bk = (u32)(key >> shift);
      }
    }
    smem_bump(hist, bk, bk != 0xffffffffu);
  }
  __syncthreads();
  for (u32 b = threadIdx.x; b < nb; b += blockDim.x) blk_counts[(i64)blockIdx.x * nb + b] = hist[b];
}

// one block per bucket: exclusive scan over the blocks' counts (in place)
__global__ void __launch_bounds__(1024) k_bk_cols(u32* blk_counts, u32 nblk, u32 nb, u64* bucket_tot) {
  const u32 b = blockIdx.x;
  __shared__ u32 w[32];
  __shared__ u32 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u32 base = 0; base < nblk; base += 1024) {
    const u32 k = base + threadIdx.x;
    const u32 v = k < nblk ? blk_counts[(i64)k * nb + b] : 0;
    u32 x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const u32 yv = __shfl_up_sync(kFull, x, o);
      if ((threadIdx.x & 31) >= o) x += yv;
    }
    if ((threadIdx.x & 31) == 31) w[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      u32 z = w[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const u32 yv = __shfl_up_sync(kFull, z, o);
        if ((int)threadIdx.x >= o) z += yv;
      }
      w[threadIdx.x] = z;
    }
    __syncthreads();
    const u32 before = (threadIdx.x >= 32 ? w[(threadIdx.x >> 5) - 1] : 0) + x - v;
    if (k < nblk) blk_counts[(i64)k * nb + b] = carry + before;
    __syncthreads();
    if (threadIdx.x == 1023) carry += before + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) bucket_tot[b] = carry;
}

// block-wide exclusive scan of nitems counters in shared memory
__device__ __forceinline__ void block_exclusive_scan(const u32* in, u32* out, u32 nitems, u32* warpsum) {
  const u32 per = (nitems + blockDim.x - 1) / blockDim.x;
  const u32 q0 = threadIdx.x * per;
  u32 run = 0;
  for (u32 t = 0; t < per; ++t) run += (q0 + t < nitems) ? in[q0 + t] : 0;
  u32 x = run;
  for (int o = 1; o < 32; o <<= 1) {
    const u32 yv = __shfl_up_sync(kFull, x, o);
    if ((threadIdx.x & 31) >= o) x += yv;
  }
  if ((threadIdx.x & 31) == 31) warpsum[threadIdx.x >> 5] = x;
  __syncthreads();
  u32 pre = x - run;
  for (u32 w = 0; w < (threadIdx.x >> 5); ++w) pre += warpsum[w];
  for (u32 t = 0; t < per; ++t) {
    if (q0 + t >= nitems) break;
    const u32 c = in[q0 + t];
    out[q0 + t] = pre;
    pre += c;
  }
  __syncthreads();
}

template <int D, typename RT>
constexpr int kStageRound = (SRec<D, RT>::kBytes <= 32) ? 2048 : 1024;

template <int D, typename RT>
__host__ __device__ constexpr size_t bk_stage_smem(u32 nb) {
  return (size_t)kStageRound<D, RT> * (SRec<D, RT>::kBytes + 4) + (size_t)3 * nb * 4;
}

template <int D, class Src>
__global__ void __launch_bounds__(512) k_bk_stage(Src src, i64 n, int shift, u32 nb, i64 chunk, const u32* blk_off,
                                                  const u64* bucket_base, const u32* __restrict__ cell0,
                                                  uint4* __restrict__ stage) {
  using RT = typename Src::RT;
  constexpr int R = kStageRound<D, RT>;
  constexpr int PER = R / 512;
  constexpr int V = SRec<D, RT>::kVec;
  extern __shared__ __align__(16) unsigned char raw[];
  uint4* recs = reinterpret_cast<uint4*>(raw);                    // [R][V]
  u32* rbk = reinterpret_cast<u32*>(recs + (size_t)R * V);        // [R] bucket of local record
  u32* gcur = rbk + R;                                            // [nb] global cursor
  u32* lcnt = gcur + nb;                                          // [nb] round counts
  u32* lst = lcnt + nb;                                           // [nb] round starts
  __shared__ u32 warpsum[32];
  for (u32 b = threadIdx.x; b < nb; b += blockDim.x)
    gcur[b] = (u32)bucket_base[b] + blk_off[(i64)blockIdx.x * nb + b];
  for (int q = threadIdx.x; q < R; q += blockDim.x) rbk[q] = 0xffffffffu;
  const i64 a0 = (i64)blockIdx.x * chunk, a1 = min(n, a0 + chunk);
  for (i64 r0 = a0; r0 < a1; r0 += R) {
    const int m = (int)min((i64)R, a1 - r0);
    for (u32 b = threadIdx.x; b < nb; b += blockDim.x) lcnt[b] = 0;
    __syncthreads();
    // all global loads of the round first (memory-level parallelism), then
    // local ranks per bucket
    u32 mykey[PER], mybk[PER], myrk[PER];
    RT myv[PER][D];
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int q = t * 512 + threadIdx.x;
      mykey[t] = q < m ? __ldcs(cell0 + r0 + q) : 0xffffffffu;
      if (q < m) src.raw(r0 + q, myv[t]);
    }
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const u32 bk = mykey[t] == 0xffffffffu ? 0xffffffffu : mykey[t] >> shift;
      mybk[t] = bk;
      myrk[t] = smem_bump(lcnt, bk, bk != 0xffffffffu);
    }
    __syncthreads();
    block_exclusive_scan(lcnt, lst, nb, warpsum);
    // records into bucket order in shared memory
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int q = t * 512 + threadIdx.x;
      if (mybk[t] == 0xffffffffu) continue;
      const u32 lpos = lst[mybk[t]] + myrk[t];
      srec_put<D, RT>(reinterpret_cast<u32*>(recs + (size_t)lpos * V), myv[t], (u32)(r0 + q));
      rbk[lpos] = mybk[t];
    }
    __syncthreads();
    // coalesced write-out: consecutive local records of one bucket go to
    // consecutive staging records
    for (int q = threadIdx.x; q < m; q += blockDim.x) {
      const u32 bk = rbk[q];
      if (bk == 0xffffffffu) continue;
      const u32 pos = gcur[bk] + (q - lst[bk]);
#pragma unroll
      for (int w = 0; w < V; ++w) stage[(i64)pos * V + w] = recs[(size_t)q * V + w];
      rbk[q] = 0xffffffffu;
    }
    __syncthreads();
    for (u32 b = threadIdx.x; b < nb; b += blockDim.x) gcur[b] += lcnt[b];
    __syncthreads();
  }
}

// A chunk = TT*kRpt staging records, kRpt per thread of a TT-thread block
// (record r0 + t*TT + tid); each thread keeps its records' slots and indices
// in registers across the passes.  k_bk_tally: 512 threads (fewer window
// clears per record), k_bk_place: 256 threads (shorter barrier chains).
constexpr int kRpt = 8;
constexpr int kTallyThreads = 512, kPlaceThreads = 256;
static_assert(kChunkRecs == kRpt * kTallyThreads, "tally chunk = records per thread x threads");

template <int D, typename RT, int TT>
__device__ __forceinline__ void load_slots(const uint4* __restrict__ stage, const GridParams& g, i64 r0, i64 r1,
                                           u32 (&key)[kRpt], u32 (&idx)[kRpt], Ctrl* ctrl) {
  constexpr int V = SRec<D, RT>::kVec;
#pragma unroll
  for (int t = 0; t < kRpt; ++t) {
    const i64 r = r0 + t * TT + threadIdx.x;
    key[t] = 0xffffffffu;
    idx[t] = 0xffffffffu;
    if (r < r1) {
      double v[D];
      bool inside;
      const u32 k = srec_slot<D, RT>(g, stage + r * V, v, idx[t], inside);
      if (inside) key[t] = k; else atomicOr(&ctrl->error, kErrMissing);
    }
  }
}

// slot range [kmin, kmax] of the chunk (block-wide)
__device__ __forceinline__ void slots_range(const u32 (&key)[kRpt], u32* kmin_s, u32* kmax_s) {
  if (threadIdx.x == 0) { *kmin_s = 0xffffffffu; *kmax_s = 0; }
  __syncthreads();
  u32 lmin = 0xffffffffu, lmax = 0;
#pragma unroll
  for (int t = 0; t < kRpt; ++t) {
    if (key[t] == 0xffffffffu) continue;
    lmin = min(lmin, key[t]);
    lmax = max(lmax, key[t]);
  }
  lmin = __reduce_min_sync(kFull, lmin);
  lmax = __reduce_max_sync(kFull, lmax);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(kmin_s, lmin);
    atomicMax(kmax_s, lmax);
  }
  __syncthreads();
}

// per chunk of staging: per-slot counts and minimum original index through
// shared-memory tallies over the chunk's slot window, then one global atomic
// pair per (chunk, slot).  cnt must be zero on entry.
template <int D, typename RT>
__global__ void __launch_bounds__(kTallyThreads) k_bk_tally(const uint4* __restrict__ stage, i64 n, u64 nslots, GridParams g,
                                                  u32* cnt, u32* minidx, Ctrl* ctrl) {
  constexpr int WIN = kTallyWin;
  extern __shared__ u32 tsm[];
  u32* lc = tsm;
  u32* mn = tsm + WIN;
  __shared__ u32 kmin_s, kmax_s;
  const i64 r0 = (i64)blockIdx.x * kChunkRecs, r1 = min(n, r0 + kChunkRecs);
  u32 key[kRpt], idx[kRpt];
  load_slots<D, RT, kTallyThreads>(stage, g, r0, r1, key, idx, ctrl);
  slots_range(key, &kmin_s, &kmax_s);
  const u32 kmin = kmin_s;
  const bool wide = kmax_s >= nslots || kmax_s - kmin >= (u32)WIN;
  const u32 span = wide ? 0 : kmax_s - kmin + 1;
  for (u32 q = threadIdx.x; q < span; q += blockDim.x) {
    lc[q] = 0;
    mn[q] = 0xffffffffu;
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < kRpt; ++t) {
    const bool valid = key[t] != 0xffffffffu;
    if (wide) {
      if (valid && key[t] < nslots) {
        atomicAdd(cnt + key[t], 1u);
        atomicMin(minidx + key[t], idx[t]);
      }
      continue;
    }
    // one atomic pair for a warp on a single slot (hot cells), else per lane
    const u32 k0 = __shfl_sync(kFull, key[t], 0);
    if (__all_sync(kFull, valid && key[t] == k0)) {
      const u32 mnv = __reduce_min_sync(kFull, idx[t]);
      if ((threadIdx.x & 31) == 0) {
        atomicAdd(lc + (k0 - kmin), 32u);
        atomicMin(mn + (k0 - kmin), mnv);
      }
    } else if (valid) {
      atomicAdd(lc + (key[t] - kmin), 1u);
      atomicMin(mn + (key[t] - kmin), idx[t]);
    }
  }
  __syncthreads();
  for (u32 q = threadIdx.x; q < span; q += blockDim.x) {
    if (!lc[q]) continue;
    atomicAdd(cnt + kmin + q, lc[q]);
    atomicMin(minidx + kmin + q, mn[q]);
  }
}

// per chunk again: one global cursor bump per (chunk, slot), shared-memory
// local ranks, SoA fp64 writes of the sorted iterate (off ends as run ends)
template <int D, typename RT>
__global__ void __launch_bounds__(kPlaceThreads) k_bk_place(const uint4* __restrict__ stage, i64 n, u64 nslots, GridParams g,
                                                  u32* off, double* __restrict__ ys, Ctrl* ctrl, u32* perm) {
  constexpr int WIN = kTallyWin;
  constexpr int V = SRec<D, RT>::kVec;
  extern __shared__ u32 cnt[];
  __shared__ u32 kmin_s, kmax_s;
  constexpr i64 kPlaceRecs = (i64)kRpt * kPlaceThreads;
  const i64 r0 = (i64)blockIdx.x * kPlaceRecs, r1 = min(n, r0 + kPlaceRecs);
  u32 key[kRpt], idx[kRpt];
  load_slots<D, RT, kPlaceThreads>(stage, g, r0, r1, key, idx, ctrl);
  slots_range(key, &kmin_s, &kmax_s);
  const u32 kmin = kmin_s;
  const bool wide = kmax_s >= nslots || kmax_s - kmin >= (u32)WIN;
  u32 pos[kRpt];
  if (!wide) {
    const u32 span = kmax_s - kmin + 1;
    for (u32 q = threadIdx.x; q < span; q += blockDim.x) cnt[q] = 0;
    __syncthreads();
#pragma unroll
    for (int t = 0; t < kRpt; ++t) pos[t] = smem_bump(cnt, key[t] - kmin, key[t] != 0xffffffffu);
    __syncthreads();
    for (u32 q = threadIdx.x; q < span; q += blockDim.x)
      if (cnt[q]) cnt[q] = atomicAdd(off + kmin + q, cnt[q]);   // now the chunk's base
    __syncthreads();
#pragma unroll
    for (int t = 0; t < kRpt; ++t)
      if (key[t] != 0xffffffffu) pos[t] += cnt[key[t] - kmin];
  } else {
#pragma unroll
    for (int t = 0; t < kRpt; ++t) {
      if (key[t] >= nslots) key[t] = 0xffffffffu;
      pos[t] = key[t] != 0xffffffffu ? atomicAdd(off + key[t], 1u) : 0u;
    }
  }
#pragma unroll
  for (int t = 0; t < kRpt; ++t) {
    if (key[t] == 0xffffffffu || pos[t] >= (u32)n) continue;
    double v[D];
    srec_coords<D, RT>(stage + (r0 + t * kPlaceThreads + threadIdx.x) * V, v);
#pragma unroll
    for (int j = 0; j < D; ++j) __stcs(ys + (i64)j * g.ld + pos[t], v[j]);
    if (perm) perm[pos[t]] = idx[t];   // sorted position -> original index
  }
}

// ------------------------------------------------------------- extraction

__device__ __forceinline__ u32 uf_root(u32* par, u32 v) {
  u32 curr = *(volatile u32*)(par + v);
  if (curr != v) {
    u32 prev = v, next;
    while (curr > (next = *(volatile u32*)(par + curr))) {
      par[prev] = next;   // path halving; benign race (parents only decrease)
      prev = curr;
      curr = next;
    }
  }
  return curr;
}

// Read-only root walk.  Used once all unions are done: a path-halving walk
// here could overwrite another thread's freshly flattened par[s] = root
// with an intermediate node.
__device__ __forceinline__ u32 uf_root_ro(const u32* par, u32 v) {
  u32 p = *(volatile const u32*)(par + v);
  while (p != v) {
    v = p;
    p = *(volatile const u32*)(par + v);
  }
  return v;
}

__device__ __forceinline__ void uf_unite(u32* par, u32 a, u32 b) {
  u32 ra = uf_root(par, a), rb = uf_root(par, b);
  while (ra != rb) {
    if (ra < rb) { const u32 t = ra; ra = rb; rb = t; }
    const u32 old = atomicCAS(par + ra, ra, rb);   // hook the larger root
    if (old == ra) return;
    ra = uf_root(par, old);
    rb = uf_root(par, rb);
  }
}

// par[s] = the first occupied lexicographically earlier neighbour with a
// smaller slot (ECL-CC style initial hooking: most unions of k_uf_link then
// find their roots already equal), else s.
template <int D, class Tab>
__global__ void k_uf_init(GridParams g, Tab tab, const u32* kp, u32* par, u32* first) {
  constexpr int M = (D == 1) ? 3 : (D == 2) ? 9 : (D == 3) ? 27 : (D == 4) ? 81 :
                    (D == 5) ? 243 : (D == 6) ? 729 : (D == 7) ? 2187 : 6561;
  const u32 k = *kp;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < k; a += stride) {
    const u32 s = tab.list[a];
    const u64 key = tab.key_of(s);
    u32 p = s;
    for (int o = 0; o < M / 2 && p == s; ++o) {
      int r = o;
      i64 delta = 0;
#pragma unroll
      for (int j = D - 1; j >= 0; --j) {
        delta += (i64)((r % 3) - 1) * (i64)g.stride[j];
        r /= 3;
      }
      u32 ns;
      if (tab.find(key + (u64)delta, ns) && ns < s) p = ns;
    }
    par[s] = p;
    first[s] = 0xffffffffu;
  }
}

template <int D, class Tab>
__global__ void k_uf_link(GridParams g, Tab tab, const u32* kp, u32* par) {
  constexpr int M = (D == 1) ? 3 : (D == 2) ? 9 : (D == 3) ? 27 : (D == 4) ? 81 :
                    (D == 5) ? 243 : (D == 6) ? 729 : (D == 7) ? 2187 : 6561;
  const u32 k = *kp;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < k; a += stride) {
    const u32 s = tab.list[a];
    const u64 key = tab.key_of(s);
    // offsets are symmetric: linking only to lexicographically later
    // neighbours (o > M/2) covers every adjacent pair once
    for (int o = M / 2 + 1; o < M; ++o) {
      int r = o;
      i64 delta = 0;
#pragma unroll
      for (int j = D - 1; j >= 0; --j) {
        delta += (i64)((r % 3) - 1) * (i64)g.stride[j];
        r /= 3;
      }
      u32 ns;
      if (tab.find(key + (u64)delta, ns) && *(volatile u32*)(par + s) != *(volatile u32*)(par + ns))
        uf_unite(par, s, ns);
    }
  }
}

// Component root per occupied cell + exact per-component count/sums
// (accumulated into the clean scratch entries `acc`, indexed by root slot).
template <int D, class Tab>
__global__ void k_uf_flatten(Tab tab, const u32* kp, u32* par, Entry<D>* acc) {
  const u32 k = *kp;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count (the group sums below are warp collectives)
  for (i64 base = (i64)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < k; base += stride) {
    const i64 a = base + lane;
    u32 r = 0xffffffffu;
    u64 w[1 + 2 * D];
#pragma unroll
    for (int q = 0; q < 1 + 2 * D; ++q) w[q] = 0;
    if (a < k) {
      const u32 s = tab.list[a];
      r = uf_root_ro(par, s);
      par[s] = r;   // only the owner writes par[s]; every other write is a root
      const Entry<D>& e = tab.ent[s];
      w[0] = e.count;
#pragma unroll
      for (int j = 0; j < D; ++j) { w[1 + j] = e.hi[j]; w[1 + D + j] = e.lo[j]; }
    }
    // cells of one component (most of a warp, for big clusters) add once
    const unsigned peers = __match_any_sync(kFull, r);
    if (__any_sync(kFull, __popc(peers) > 1)) {
#pragma unroll
      for (int kk = 0; kk < 5; ++kk) {
        const unsigned src = __fns(peers, lane, (1 << kk) + 1);
        const int from = src < 32 ? (int)src : lane;
#pragma unroll
        for (int q = 0; q < 1 + 2 * D; ++q) {
          const u64 o = __shfl_sync(kFull, w[q], from);
          if (src < 32) w[q] += o;
        }
      }
    }
    if (r == 0xffffffffu || lane != __ffs(peers) - 1) continue;
    Entry<D>* c = acc + r;
    atomicAdd(&c->count, w[0]);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      atomicAdd(&c->hi[j], w[1 + j]);
      atomicAdd(&c->lo[j], w[1 + D + j]);
    }
  }
}

// First appearance: minimum original point index per component
// (modeseek.py:262-265).  par[] is flat here (k_uf_flatten), so the
// component of a cell is one load; lanes sharing a component are reduced
// with match_any + reduce_min before the single atomicMin.
template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_first(const double* __restrict__ y, i64 n, GridParams g, Tab tab,
                                                    const u32* par, u32* first, const u32* perm, Ctrl* ctrl,
                                                    u32 offset) {
  const int lane = threadIdx.x & 31;
  const i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const i64 nwarps = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 base = warp * 32; base < n; base += nwarps * 32) {
    const i64 i = base + lane;
    u32 r = 0xffffffffu, idx = 0xffffffffu;
    if (i < n) {
      double v[D];
#pragma unroll
      for (int j = 0; j < D; ++j) v[j] = y[(i64)j * g.ld + i];
      bool inside;
      const u64 key = pack_key<D>(g, v, inside);
      u32 s;
      if (inside && tab.find(key, s)) {
        r = par[s];
        idx = (perm ? perm[i] : (u32)i) + offset;
      } else {
        atomicOr(&ctrl->error, kErrMissing);
      }
    }
    const unsigned peers = __match_any_sync(kFull, r);
    const u32 best = __reduce_min_sync(peers, idx);
    if (r != 0xffffffffu && lane == __ffs(peers) - 1) atomicMin(first + r, best);
  }
}

template <int D, class Tab>
__global__ void k_roots(Tab tab, const u32* kp, const u32* par, const u32* first, u32* roots,
                        u32* root_first, u32* nroots) {
  const u32 k = *kp;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < k; a += stride) {
    const u32 s = tab.list[a];
    if (par[s] == s) {
      const u32 idx = atomicAdd(nroots, 1u);
      roots[idx] = s;
      root_first[idx] = first[s];
    }
  }
}

// rank[] for roots (host-sorted by first appearance) -> rankmap[slot];
// modes = exact component sum / count (modeseek.py:268-271).
template <int D>
__global__ void k_modes(GridParams g, const u32* roots, const u32* ranks, u32 nr, u32* rankmap,
                        Entry<D>* acc, double* modes) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < nr; a += stride) {
    const u32 r = roots[a];
    const u32 rk = ranks[a];
    rankmap[r] = rk;
    Entry<D>* c = acc + r;
    const double cnt = (double)c->count;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const i128 s = (((i128)(i64)c->hi[j]) << 32) + (i128)c->lo[j];
      modes[(i64)rk * D + j] = __ddiv_rn(i128_to_double(s, -g.qexp[j]), cnt);
      c->hi[j] = 0;
      c->lo[j] = 0;
    }
    c->count = 0;
  }
}

template <int D, class Tab>
__global__ void __launch_bounds__(kThreads) k_labels(const double* __restrict__ y, i64 n, GridParams g, Tab tab,
                                                     const u32* par, const u32* rankmap, const u32* perm,
                                                     i64* labels) {
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double v[D];
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] = y[(i64)j * g.ld + i];
    bool inside;
    const u64 key = pack_key<D>(g, v, inside);
    u32 s = 0;
    if (inside) tab.find(key, s);
    const u32 r = par[s];
    const i64 idx = perm ? (i64)perm[i] : i;
    labels[idx] = (i64)rankmap[r];
  }
}

// Clear a table's occupied entries (and keys) and reset its count.
template <int D, class Tab>
__global__ void k_clear(Tab tab, u32* kp) {
  const u32 k = *kp;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < k; a += stride) {
    const u32 s = tab.list[a];
    Entry<D>* e = tab.ent + s;
    e->count = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) { e->hi[j] = 0; e->lo[j] = 0; }
    if constexpr (!Tab::kDense) tab.keys[s] = kEmpty;
  }
}

__global__ void k_reset_count(u32* kp) { *kp = 0; }

// Occupied-cell dump for build_cell_tables / neighbour stats (grid.py:193, 230).
template <int D, class Tab>
__global__ void k_dump(GridParams g, Tab tab, const u32* kp, u64* keys_out, i64* counts_out,
                       double* sums_out, i64* ncounts_out, double* nsums_out, const double* rs = nullptr) {
  const u32 k = *kp;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < k; a += stride) {
    const u32 s = tab.list[a];
    const u64 key = tab.key_of(s);
    keys_out[a] = key;
    const Entry<D>& e = tab.ent[s];
    counts_out[a] = (i64)e.count;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const i128 v = (((i128)(i64)e.hi[j]) << 32) + (i128)e.lo[j];
      sums_out[a * D + j] = rs ? rs[(i64)s * D + j] : i128_to_double(v, -g.qexp[j]);
    }
    if (ncounts_out) {
      u64 cnt;
      if (rs) {
        double sum[D];
        neighbourhood_sum_rs<D>(g, tab, rs, key, cnt, sum);
#pragma unroll
        for (int j = 0; j < D; ++j) nsums_out[a * D + j] = sum[j];
      } else {
        i128 sum[D];
        neighbourhood_sum<D>(g, tab, key, cnt, sum);
#pragma unroll
        for (int j = 0; j < D; ++j) nsums_out[a * D + j] = i128_to_double(sum[j], -g.qexp[j]);
      }
      ncounts_out[a] = (i64)cnt;
    }
  }
}

}  // namespace gs
