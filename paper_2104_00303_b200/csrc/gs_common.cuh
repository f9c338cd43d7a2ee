// gridshift-b200: shared device definitions.
//
// Numerics contract:
//   * binning is IEEE fp64 floor(y / h)  (reference grid.py:81; never y*(1/h))
//   * per-cell coordinate sums are EXACT: every coordinate is mapped to a
//     signed fixed-point integer v = rne(y * 2^s_j), |v| < 2^61, and
//     accumulated as (sum of v>>32, sum of v&0xffffffff) in two 64-bit
//     integer words, so the total is order-independent and bit-reproducible
//     (reference grid.py:186-187 sums sequentially in fp64; only keys and
//     counts are a bit-exact contract, sums need to stay within 1e-9*h)
//   * the 3^d neighbourhood sum is formed exactly in __int128 and rounded
//     once to fp64 (correct rounding), then divided: y' = S / C
//     (reference modeseek.py:109)
//   * per-point movement norms are summed in 128-bit fixed point, so the
//     convergence value is independent of thread scheduling.
#pragma once

#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#ifndef GS_MAXD
#define GS_MAXD 8
#endif

namespace gs {

typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;
typedef unsigned char u8;
typedef __int128 i128;
typedef unsigned __int128 u128;

constexpr u64 kEmpty = ~0ull;

// Lattice + quantisation parameters for one engine run (passed by value).
struct GridParams {
  double h;
  int d;
  int movement_exp;        // norms are quantised with 2^(96 - movement_exp)
  i64 base[GS_MAXD];       // key origin per axis (= lowest admissible cell - 1)
  i64 lo[GS_MAXD];         // admissible cell box, inclusive
  i64 hi[GS_MAXD];
  u64 stride[GS_MAXD];     // row-major strides, last axis fastest (grid.py:153-157)
  double qscale[GS_MAXD];  // 2^s_j : fixed-point scale per axis
  int qexp[GS_MAXD];       // s_j
  u64 nkeys;               // prod of extents
  u64 mask;                // hash mask (cap - 1) or 0 for dense tables
  i64 ld;                  // SoA leading dimension of the iterate (n rounded up to 128)
  double inv_h;            // fl(1 / h), for cell_of_fast
  int pad_;                // (unused; keeps the layout)
};

// Device-resident loop control.  One per context.
struct Ctrl {
  int done;                // set by the shift kernel when movement < eta
  int iters;               // iterations executed
  int error;               // bit flags, see kErr*
  int pad;
  u32 k[2];                // occupied-cell count of the two table buffers
  u32 blocks_done;         // last-block detection for the movement reduction
  u32 agg_done;            // last-block detection in k_agg
  u32 nruns;               // initial cells (runs) after the spatial sort
  u32 pad3;
};

// Kernels of iteration t skip once the run stopped at an earlier iteration:
// `done` holds (stopping iteration + 1).  The table chain may run one
// iteration ahead of the shifts (side stream), so a plain flag would let the
// shift of iteration t cancel the k_derive of the same iteration.
__device__ __forceinline__ bool stopped_before(const Ctrl* c, int t) {
  const int d = *(volatile const int*)&c->done;
  return d != 0 && d <= t;
}

// Block-uniform form: `done` can flip while a side-stream kernel runs, and a
// block whose warps disagreed would run its shared-memory phases half-staffed.
__device__ __forceinline__ bool block_stopped_before(const Ctrl* c, int t) {
  __shared__ int stop;
  if (threadIdx.x == 0) stop = stopped_before(c, t);
  __syncthreads();
  return stop != 0;
}

constexpr int kErrOutOfBox = 1;     // an iterate left the admissible lattice box
constexpr int kErrTableFull = 2;    // hash table overflow (cannot happen at load <= 1/2)
constexpr int kErrNonFinite = 4;    // NaN/inf in input
constexpr int kErrLattice = 8;      // |floor(y/h)| >= 2^62 (grid.py:82-84)
constexpr int kErrMissing = 16;     // a lookup missed a cell that must exist

// One occupied cell: count plus split fixed-point sums.
template <int D>
struct Entry {
  u64 count;
  u64 hi[D];   // sum of (v >> 32), two's complement
  u64 lo[D];   // sum of (v & 0xffffffff)
};

__host__ __device__ inline u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// x * 2^k, rounded once like ldexp: a multiply by the power of two when
// 2^k is a normal double (IEEE multiply rounds exactly as ldexp does), the
// library ldexp otherwise.
__host__ __device__ inline double scale2(double x, int k) {
  if (k >= -1022 && k <= 1023) {
    u64 bits = (u64)(k + 1023) << 52;
    double p;
    memcpy(&p, &bits, sizeof p);
    return x * p;
  }
  return ldexp(x, k);
}

// Correctly rounded (round-to-nearest-even) value of v * 2^e as a double.
__host__ __device__ inline double i128_to_double(i128 v, int e) {
  if (v == 0) return 0.0;
  const bool neg = v < 0;
  u128 u = neg ? (u128)(-v) : (u128)v;
  const u64 hw = (u64)(u >> 64);
  const u64 lw = (u64)u;
  int nb;
#ifdef __CUDA_ARCH__
  nb = hw ? 128 - __clzll((i64)hw) : 64 - __clzll((i64)lw);
#else
  nb = hw ? 128 - __builtin_clzll(hw) : 64 - __builtin_clzll(lw);
#endif
  u64 m;
  int sh = 0;
  if (nb <= 53) {
    m = lw;
  } else {
    sh = nb - 53;
    m = (u64)(u >> sh);
    const u128 rem = u & ((((u128)1) << sh) - 1);
    const u128 half = ((u128)1) << (sh - 1);
    if (rem > half || (rem == half && (m & 1ull))) {
      m += 1;
      if (m == (1ull << 53)) { m >>= 1; sh += 1; }
    }
  }
  double r = scale2((double)m, e + sh);
  return neg ? -r : r;
}

__host__ __device__ inline double u128_to_double(u128 u, int e) {
  if (u == 0) return 0.0;
  // |u| < 2^127 by construction, so the signed path is exact.
  return i128_to_double((i128)u, e);
}

// Fixed-point image of one coordinate: rne(y * 2^s), |result| < 2^61.
__device__ __forceinline__ i64 to_fixed(double y, double qscale) {
  return __double2ll_rn(__dmul_rn(y, qscale));
}

// 128-bit fixed-point image of a non-negative norm: rne(m * 2^(96-E)).
__device__ __forceinline__ u128 norm_to_fixed(double m, int movement_exp) {
  // split at 2^48 so both halves convert exactly
  const double a = scale2(m, 48 - movement_exp);     // < 2^48
  const double ia = floor(a);
  const double r = __dsub_rn(a, ia);               // exact
  const u64 hi = (u64)ia;
  const u64 lo = (u64)__double2ll_rn(scale2(r, 48));
  return (((u128)hi) << 48) + (u128)lo;
}

// Floor of the IEEE quotient fl(y / h), as an integer-valued double
// (grid.py:81 `np.floor(data / h)`).
__device__ __forceinline__ double cell_of(double y, double h) {
  return floor(__ddiv_rn(y, h));
}

// Same value, cheaper: q = fl(y * fl(1/h)) is within |q| * 2^-51 of
// Q = fl(y / h) (two roundings of 2^-53 each plus the reciprocal's), so
// unless an integer lies within that distance of q, floor(q) == floor(Q).
// Points near a cell face (and all non-finite cases) take the exact divide.
__device__ __forceinline__ double cell_of_fast(double y, double h, double inv_h) {
  const double q = __dmul_rn(y, inv_h);
  const double f = floor(q);
  const double r = __dsub_rn(q, f);   // exact: the fraction of a double
  const double tol = fmax(fabs(q), 1.0) * 0x1p-50;
  if (r > tol && r < 1.0 - tol) return f;
  return floor(__ddiv_rn(y, h));
}

__device__ __forceinline__ u64 hash_key(u64 k) { return mix64(k ^ 0x2545F4914F6CDD1Dull); }

}  // namespace gs
