// gridshift-b200: window tracker (Algorithm 3 of the paper; reference
// track.py:147-205) as one persistent CTA that walks the whole frame
// sequence resident in HBM.
//
// Per frame: up to `max_iters` re-centring steps.  Each step tests every
// window pixel's colour cell (floor(c/h) per channel, track.py:168 via
// bin_points grid.py:81) against the bin set B held as a bitmap over the
// colour lattice [0, L)^3 in shared memory, and reduces the count and the
// integer x / y sums of the hits (track.py:173: the mean of integer pixel
// coordinates is exact).  The centre is clamped (track.py:74-77) and the
// loop stops once it moves less than `tol` (track.py:176-179).  No hits
// freezes the window and flags the object lost (track.py:170-172).  With
// update_bins, B <- cells(window) & N(B) unless empty (track.py:181-186);
// N(B) is the 3x3x3 dilation of the bitmap (track.py:138-144).
#pragma once

#include "gs_common.cuh"

namespace gs {

constexpr int kTrackThreads = 1024;

struct TrackParams {
  int n_frames, height, width;
  int w, hp;               // window extents
  int L;                   // colour cells per axis
  int update_bins;
  int max_iters;
  double tol;
  double cx0, cy0;
  int words;               // bitmap words (L^3 / 32 rounded up)
  int init_matches;
};

__device__ __forceinline__ void track_rect(double cx, double cy, int w, int hp, int fw, int fh,
                                           int& x0, int& y0, int& x1, int& y1) {
  // Window.rect, track.py:43-49
  int a = (int)floor(__dadd_rn(__dsub_rn(cx, w / 2.0), 0.5));
  int b = (int)floor(__dadd_rn(__dsub_rn(cy, hp / 2.0), 0.5));
  a = min(max(a, 0), max(fw - w, 0));
  b = min(max(b, 0), max(fh - hp, 0));
  x0 = a;
  y0 = b;
  x1 = min(a + w, fw);
  y1 = min(b + hp, fh);
}

// bitmaps: B (current bins), S (seen cells), N scratch; global memory so
// large lattices (small h) work; for the common h the whole set is a few KB
// and stays in L1.
__global__ void __launch_bounds__(kTrackThreads, 1)
k_track(const unsigned char* __restrict__ frames, TrackParams p, const int* __restrict__ lut_g,
        u32* bmB, u32* bmS, double* cx_out, double* cy_out, int* lost_out, long long* matches_out,
        long long* nbins_out, u32* bm_hist) {
  __shared__ int lut[256];
  __shared__ long long red[3][kTrackThreads / 32];
  __shared__ double s_cx, s_cy;
  __shared__ int s_lost, s_any;
  __shared__ long long s_cnt, s_sx, s_sy;
  const int tid = threadIdx.x;
  for (int i = tid; i < 256; i += blockDim.x) lut[i] = lut_g[i];
  if (tid == 0) {
    s_cx = p.cx0;
    s_cy = p.cy0;
    s_lost = 0;
  }
  __syncthreads();
  const int L = p.L;
  const size_t frame_bytes = (size_t)p.height * p.width * 3;
  for (int f = 1; f < p.n_frames; ++f) {
    if (s_lost) {
      // frozen rows after the object left (track.py:201-204)
      if (tid == 0) {
        cx_out[f] = s_cx;
        cy_out[f] = s_cy;
        lost_out[f] = 1;
        matches_out[f] = 0;
        nbins_out[f] = nbins_out[f - 1];
      }
      if (bm_hist)
        for (int q = tid; q < p.words; q += blockDim.x) bm_hist[(size_t)f * p.words + q] = bmB[q];
      continue;
    }
    const unsigned char* fr = frames + (size_t)f * frame_bytes;
    double cx = s_cx, cy = s_cy;
    long long matches = 0;
    bool lost = false;
    for (int it = 0; it < p.max_iters; ++it) {
      int x0, y0, x1, y1;
      track_rect(cx, cy, p.w, p.hp, p.width, p.height, x0, y0, x1, y1);
      const int ww = x1 - x0;
      const int npx = ww * (y1 - y0);
      long long c = 0, sx = 0, sy = 0;
      for (int q = tid; q < npx; q += blockDim.x) {
        const int ry = q / ww, rx = q - ry * ww;
        const unsigned char* px = fr + ((size_t)(y0 + ry) * p.width + (x0 + rx)) * 3;
        const int code = (lut[px[0]] * L + lut[px[1]]) * L + lut[px[2]];
        if ((bmB[code >> 5] >> (code & 31)) & 1u) {
          ++c;
          sx += x0 + rx;
          sy += y0 + ry;
        }
      }
      for (int o = 16; o; o >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, o);
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
      }
      if ((tid & 31) == 0) {
        red[0][tid >> 5] = c;
        red[1][tid >> 5] = sx;
        red[2][tid >> 5] = sy;
      }
      __syncthreads();
      if (tid == 0) {
        long long tc = 0, tx = 0, ty = 0;
        for (int wq = 0; wq < (int)(blockDim.x >> 5); ++wq) {
          tc += red[0][wq];
          tx += red[1][wq];
          ty += red[2][wq];
        }
        s_cnt = tc;
        s_sx = tx;
        s_sy = ty;
      }
      __syncthreads();
      matches = s_cnt;
      if (matches == 0) {
        lost = true;
        break;
      }
      double nx = __ddiv_rn((double)s_sx, (double)matches);
      double ny = __ddiv_rn((double)s_sy, (double)matches);
      // _clamp_center, track.py:74-77
      nx = fmin(fmax(nx, p.w / 2.0), p.width - p.w / 2.0);
      ny = fmin(fmax(ny, p.hp / 2.0), p.height - p.hp / 2.0);
      const double moved = hypot(__dsub_rn(nx, cx), __dsub_rn(ny, cy));
      cx = nx;
      cy = ny;
      __syncthreads();
      if (moved < p.tol) break;
    }
    if (lost) {
      if (tid == 0) {
        s_lost = 1;
        cx_out[f] = s_cx;   // window frozen at its incoming position
        cy_out[f] = s_cy;
        lost_out[f] = 1;
        matches_out[f] = 0;
        nbins_out[f] = nbins_out[f - 1];
      }
      if (bm_hist)
        for (int q = tid; q < p.words; q += blockDim.x) bm_hist[(size_t)f * p.words + q] = bmB[q];
      __syncthreads();
      continue;
    }
    if (p.update_bins) {
      int x0, y0, x1, y1;
      track_rect(cx, cy, p.w, p.hp, p.width, p.height, x0, y0, x1, y1);
      const int ww = x1 - x0;
      const int npx = ww * (y1 - y0);
      for (int q = tid; q < p.words; q += blockDim.x) bmS[q] = 0;
      __syncthreads();
      for (int q = tid; q < npx; q += blockDim.x) {
        const int ry = q / ww, rx = q - ry * ww;
        const unsigned char* px = fr + ((size_t)(y0 + ry) * p.width + (x0 + rx)) * 3;
        const int code = (lut[px[0]] * L + lut[px[1]]) * L + lut[px[2]];
        atomicOr(bmS + (code >> 5), 1u << (code & 31));
      }
      if (tid == 0) s_any = 0;
      __syncthreads();
      // fresh = seen & N(B)
      int any = 0;
      for (int q = tid; q < p.words; q += blockDim.x) {
        u32 seen = bmS[q], keep = 0;
        while (seen) {
          const int bit = __ffs(seen) - 1;
          seen &= seen - 1;
          const int code = q * 32 + bit;
          const int a = code / (L * L), b = (code / L) % L, cc = code % L;
          bool hit = false;
          for (int da = -1; da <= 1 && !hit; ++da)
            for (int db = -1; db <= 1 && !hit; ++db)
              for (int dc = -1; dc <= 1 && !hit; ++dc) {
                const int A = a + da, Bq = b + db, C = cc + dc;
                if (A < 0 || Bq < 0 || C < 0 || A >= L || Bq >= L || C >= L) continue;
                const int nc = (A * L + Bq) * L + C;
                hit = (bmB[nc >> 5] >> (nc & 31)) & 1u;
              }
          if (hit) keep |= 1u << bit;
        }
        bmS[q] = keep;
        any |= keep != 0;
      }
      if (any) atomicOr(&s_any, 1);
      __syncthreads();
      if (s_any) {
        for (int q = tid; q < p.words; q += blockDim.x) bmB[q] = bmS[q];
      }
      __syncthreads();
    }
    // popcount of B for the row (+ the row's bin set)
    long long nb = 0;
    for (int q = tid; q < p.words; q += blockDim.x) {
      nb += __popc(bmB[q]);
      if (bm_hist) bm_hist[(size_t)f * p.words + q] = bmB[q];
    }
    for (int o = 16; o; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
    if ((tid & 31) == 0) red[0][tid >> 5] = nb;
    __syncthreads();
    if (tid == 0) {
      long long t = 0;
      for (int wq = 0; wq < (int)(blockDim.x >> 5); ++wq) t += red[0][wq];
      s_cx = cx;
      s_cy = cy;
      cx_out[f] = cx;
      cy_out[f] = cy;
      lost_out[f] = 0;
      matches_out[f] = matches;
      nbins_out[f] = t;
    }
    __syncthreads();
  }
}

}  // namespace gs
