// nufft.cu -- SAR_GRID_NUFFT (reading R19, FGG-NUFFT of P:239-242): Gaussian
// gridding of the compensated samples from their true positions + fine FFTs.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace sark {
namespace {

// --------------------------------------------------------- NUFFT mode ----
// SAR_GRID_NUFFT (reading R19, FGG-NUFFT of P:239-242).  K1n: one CTA per
// (16-wide k chunk, fine row jy of the 2ny x 2nx oversampled grid, frame).
// For each (pair, pose row) that can reach the fine row (host-built list) the
// CTA stages the pose row's samples rotated by e^{+j k beta} (Eq. (11)) and
// weighted by the row's Gaussian y-weight, plus each pose's x-weights; then
// every thread gathers into the fine-grid cells it owns (deterministic, no
// atomics).  Finally the fine row is transformed along x (N = 2nx), cropped
// to |a_s| < nx/2 and deconvolved by 1/Phi_x: Wh[f][jy][a][k].
// K2n: y-FFT over the 2ny fine rows, crop to |b_s| < ny/2, 1/Phi_y: W0.
constexpr int K1N_WT = 14;      // taps per axis: 2W + 2 with W = 6
constexpr int K1N_PCH = 256;    // poses staged at a time
constexpr int K1N_KC = 4;       // k values per CTA
constexpr int K1N_NT = 512;
template <int RX>
constexpr int k1n_br() { return RX >= 1024 ? 4 : 8; }   // fine rows per band (matches plan.cpp)

// One CTA = (k chunk of 4, band of BR fine rows, frame).  Thread (row r, k q,
// segment) owns the fine cells [seg*L, seg*L + L) x (r, q) in registers.  For
// each candidate (pair, pose row): stage the row's samples in fine-x order
// (host permutation) rotated by e^{+j k beta}, with each pose's x-weights and
// its y-weights for the band's rows; then every thread sweeps the sorted poses
// over its columns (positions may wrap by +-RX, reading R6).
template <int RX>
__global__ void __launch_bounds__(K1N_NT, 1) k1n_spread_xfft(const __grid_constant__ SarDeviceView v,
                                                             const float2 *__restrict__ s) {
  constexpr int BR = k1n_br<RX>();
  constexpr int CB = BR * K1N_KC;              // (row, k) pairs = FFT columns
  constexpr int SEGS = K1N_NT / CB;            // threads per (row, k)
  constexpr int L = RX / SEGS;                 // fine columns per thread
  extern __shared__ __align__(16) unsigned char smn[];
  const int npx = v.npx, nk = v.nk, W = v.nu_w;
  const int pch = npx < K1N_PCH ? npx : K1N_PCH;
  float2 *sval = reinterpret_cast<float2 *>(smn);                     // [pch][KC] staged samples
  float *wx = reinterpret_cast<float *>(sval + (size_t)pch * K1N_KC);  // [pch][WT]
  float *wyb = wx + (size_t)pch * K1N_WT;                             // [pch][BR]
  int *x0s = reinterpret_cast<int *>(wyb + (size_t)pch * BR);          // [pch] first tap column (no wrap)
  float2 *tile = reinterpret_cast<float2 *>(smn);                     // [RX][CB] (after the gather)
  __shared__ float2 twx[RX];
  const int tid = threadIdx.x;
  const int pair_idx = tid / SEGS, seg = tid - pair_idx * SEGS;
  const int r = pair_idx / K1N_KC, q = pair_idx - r * K1N_KC;
  const int c0 = seg * L;
  const int kc = blockIdx.x, band = blockIdx.y, f = blockIdx.z;
  const int RY = 2 * v.ny, NB = (RY + BR - 1) / BR;
  for (int i = tid; i < RX; i += K1N_NT) {
    float sn, cs;
    sincospif(-2.0f * (float)i / (float)RX, &sn, &cs);   // twiddles of the fine x-FFT
    twx[i] = make_float2(cs, sn);
  }
  const float inv2s2 = 0.5f / v.nu_s2;
  float2 acc[L];
#pragma unroll
  for (int m = 0; m < L; ++m) acc[m] = make_float2(0.f, 0.f);
  const int e0 = v.nu_off[f * NB + band], e1 = v.nu_off[f * NB + band + 1];
  for (int e = e0; e < e1; ++e) {
    const int code = __ldg(v.nu_cand + e);
    const int pr = code >> 16, iy = code & 0xffff;
    const int t = pr / v.nr, rr = pr - t * v.nr;
    const int jx2 = 2 * v.jx[pr];
    const size_t prow = (size_t)f * v.P + (size_t)iy * npx;
    const float2 *sg = s + (((size_t)(f * v.nt + t) * v.nr + rr) * v.P + (size_t)iy * npx) * nk;
    const float bp = v.no_comp ? 0.f : v.bpair[f * v.npair + pr];
    for (int p0 = 0; p0 < npx; p0 += K1N_PCH) {
      const int pn = npx - p0 < K1N_PCH ? npx - p0 : K1N_PCH;
      __syncthreads();   // the previous gather is done before the stage is rewritten
      for (int idx = tid; idx < pn * K1N_KC; idx += K1N_NT) {
        const int il = idx / K1N_KC, qq = idx - il * K1N_KC;
        const int ix = __ldg(v.nu_perm + prow + p0 + il);
        const int kq = kc * K1N_KC + qq;
        float2 val = make_float2(0.f, 0.f);
        if (kq < nk) {
          val = __ldcs(sg + (size_t)ix * nk + kq);
          if (!v.no_comp) {
            float turns = (__ldg(v.apose + prow + ix) + bp) * __ldg(v.kturn + kq);
            turns -= rintf(turns);
            float sn, cs;
            __sincosf(turns * 6.28318530717958647692f, &sn, &cs);
            val = cmul(val, make_float2(cs, sn));
          }
        }
        sval[idx] = val;
        if (qq == 0) {
          const float xf = (float)(2 * ix) + __ldg(v.nu_du + prow + ix);
          const int xb = (int)floorf(xf) - W;
          x0s[il] = xb + jx2;
#pragma unroll
          for (int tt = 0; tt < K1N_WT; ++tt) {
            const float dx = (float)(xb + tt) - xf;
            wx[il * K1N_WT + tt] = fabsf(dx) <= (float)W ? __expf(-dx * dx * inv2s2) : 0.f;
          }
          const float vf = (float)(2 * (iy + v.jy[pr])) + __ldg(v.nu_dv + prow + ix);
#pragma unroll
          for (int b = 0; b < BR; ++b) {
            float d = (float)(band * BR + b) - vf;
            d -= (float)RY * rintf(d / (float)RY);         // periodic fine rows (reading R6)
            wyb[il * BR + b] = fabsf(d) <= (float)W ? __expf(-d * d * inv2s2) : 0.f;
          }
        }
      }
      __syncthreads();
      // gather over the x-sorted poses: cell c gets tap c - x0 of the poses
      // with x0 <= c <= x0 + WT - 1, for the aliases c, c - RX, c + RX
      const int xlo = x0s[0], xhi = x0s[pn - 1] + K1N_WT - 1;
#pragma unroll
      for (int wrap = -1; wrap < 2; ++wrap) {
        const int cs = c0 + wrap * RX, ce = cs + L - 1;
        if (ce < xlo || cs > xhi) continue;
        // first pose whose footprint reaches cs (binary search, x0 ascending)
        int lo = 0, hi = pn;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (x0s[mid] + K1N_WT - 1 < cs) lo = mid + 1;
          else hi = mid;
        }
        for (int pp = lo; pp < pn; ++pp) {
          const int x0 = x0s[pp];
          if (x0 > ce) break;
          const float wyv = wyb[pp * BR + r];
          if (wyv == 0.f) continue;
          const float2 val = sval[pp * K1N_KC + q];
          const float2 vw = make_float2(val.x * wyv, val.y * wyv);
#pragma unroll
          for (int m = 0; m < L; ++m) {
            const int tt = cs + m - x0;
            if (tt >= 0 && tt < K1N_WT) {
              const float w = wx[pp * K1N_WT + tt];
              acc[m].x = fmaf(w, vw.x, acc[m].x);
              acc[m].y = fmaf(w, vw.y, acc[m].y);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // the band's fine rows -> x-FFT (N = RX) over CB columns, crop, deconvolve
#pragma unroll
  for (int m = 0; m < L; ++m) tile[(c0 + m) * CB + pair_idx] = acc[m];
  __syncthreads();
  const int nx = v.nx;
  const int kmax = nk - kc * K1N_KC;
  sarfft2::fft<RX, CB, CB, K1N_NT, -1, 0, false>(
      tile, twx, tid, [&](int c, int n) { return tile[n * CB + c]; }, [] {},
      [&](int c, int n, float2 x) {
        const int as = n < RX / 2 ? n : n - RX;
        const int rb = c / K1N_KC, qb = c - rb * K1N_KC;
        const int jyf = band * BR + rb;
        if (qb < kmax && jyf < RY && as >= -nx / 2 && as < nx / 2) {
          const int a = as < 0 ? as + nx : as;
          const float d = __ldg(v.nu_decx + a);
          v.wh[((size_t)(f * RY + jyf) * nx + a) * (size_t)nk + kc * K1N_KC + qb] = make_float2(x.x * d, x.y * d);
        }
      });
}

template <int RY>
__global__ void __launch_bounds__(sarfft2::nt_fft<RY, KC>()) k2n_yfft_crop(const __grid_constant__ SarDeviceView v) {
  constexpr int NT = sarfft2::nt_fft<RY, KC>();
  extern __shared__ __align__(16) float2 tly[];   // [RY][16]
  __shared__ float2 twy[RY];
  const int tid = threadIdx.x;
  const int kc = blockIdx.x, a = blockIdx.y, f = blockIdx.z;
  const int nx = v.nx, nk = v.nk, ny = v.ny;
  for (int i = tid; i < RY; i += NT) {
    float sn, cs;
    sincospif(-2.0f * (float)i / (float)RY, &sn, &cs);
    twy[i] = make_float2(cs, sn);
  }
  const float2 *src = v.wh + ((size_t)f * RY * nx + a) * (size_t)nk + kc * KC;
  const size_t row = (size_t)nx * nk;
  const int cmax = nk - kc * KC;
  for (int i = tid; i < RY * KC; i += NT) {
    const int n = i / KC, c = i - n * KC;
    tly[i] = c < cmax ? __ldcs(src + (size_t)n * row + c) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  float2 *dst = v.w0 + ((size_t)f * ny * nx + a) * (size_t)nk + kc * KC;
  sarfft2::fft<RY, KC, KC, NT, -1, 0, false>(
      tly, twy, tid, [&](int c, int n) { return tly[n * KC + c]; }, [] {},
      [&](int c, int n, float2 x) {
        const int bs = n < RY / 2 ? n : n - RY;
        if (c < cmax && bs >= -ny / 2 && bs < ny / 2) {
          const int b = bs < 0 ? bs + ny : bs;
          const float d = __ldg(v.nu_decy + b);
          dst[(size_t)b * row + c] = make_float2(x.x * d, x.y * d);
        }
      });
}


}  // namespace

cudaError_t launch_nufft(const SarDeviceView &v, const float2 *data, cudaStream_t s) {
  const int nchunk = (v.nk + KC - 1) / KC;
  {
    const int pch = v.npx < K1N_PCH ? v.npx : K1N_PCH;
    switch (2 * v.nx) {
#define X(N)                                                                                        \
  case N: {                                                                                         \
    constexpr int BR = k1n_br<N>();                                                                 \
    const size_t stage = (size_t)pch * (K1N_KC * sizeof(float2) + (K1N_WT + BR) * sizeof(float) + sizeof(int)); \
    const size_t tile = (size_t)N * BR * K1N_KC * sizeof(float2);                                   \
    const size_t smem = stage > tile ? stage : tile;                                                \
    dim3 grid((v.nk + K1N_KC - 1) / K1N_KC, (2 * v.ny + BR - 1) / BR, v.F);                          \
    cudaError_t e = cudaFuncSetAttribute(k1n_spread_xfft<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                 \
    k1n_spread_xfft<N><<<grid, K1N_NT, smem, s>>>(v, data);                                          \
    e = cudaGetLastError();                                                                         \
    if (e != cudaSuccess) return e;                                                                 \
    break;                                                                                          \
  }
      X(64) X(128) X(256) X(512) X(1024)
#undef X
      default:
        return cudaErrorInvalidValue;
    }
  }
  dim3 grid(nchunk, v.nx, v.F);
  switch (2 * v.ny) {
#define X(N)                                                                                         \
  case N: {                                                                                          \
    const size_t smem = (size_t)N * KC * sizeof(float2);                                             \
    cudaError_t e = cudaFuncSetAttribute(k2n_yfft_crop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                  \
    k2n_yfft_crop<N><<<grid, sarfft2::nt_fft<N, KC>(), smem, s>>>(v);                                \
    return cudaGetLastError();                                                                       \
  }
    X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)
#undef X
  }
  return cudaErrorInvalidValue;
}


}  // namespace sark
