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
// SAR_GRID_NUFFT (reading R19, FGG-NUFFT of P:239-242): K1s spreads the
// compensated samples onto the 2ny x 2nx fine grid, the mid-axis FFT kernel
// transforms the fine rows along x, and K2n transforms along y, crops to the
// kept frequencies and deconvolves by 1/(Phi_x Phi_y) into W0.
// K1s: the spread as a k-parallel gather.  One CTA = (4 x 8 block of fine
// cells, frame, chunk of NT wavenumbers); thread = wavenumber k, so every
// sample read is a coalesced run along k and the 32 cell accumulators live in
// registers (deterministic, no atomics).  For each host-listed entry (virtual
// element within W of the block, reading R19) the CTA stages its 32 Gaussian
// weights phi(j - U) phi(i - V) (4 threads per entry, one fine row each);
// then every thread rotates its sample by e^{+j k beta} (Eq. (11)) and
// accumulates it into the 32 cells with paired-fp32 FMAs.  The block's cells
// are written once, [F][2ny][2nx][nk]; the fine x-FFT follows (launch_mid).
constexpr int SP_CELLS = SAR_SP_BX * SAR_SP_BY;
template <int NT, int KPT>
__global__ void __launch_bounds__(NT, (KPT == 1 ? 1024 : 512) / NT) k1s_spread(const __grid_constant__ SarDeviceView v,
                                                          const float2 *__restrict__ s) {
  constexpr int CH = NT / SAR_SP_BY;   // entries staged per round (one thread per weight row)
  constexpr int U = 4 / KPT;           // entries whose samples are loaded ahead
  constexpr int KB = NT * KPT;         // wavenumbers per CTA
  __shared__ float4 ent[CH];
  __shared__ __align__(16) float wt[CH][SP_CELLS];
  const int tid = threadIdx.x;
  const int nk = v.nk;
  const int nkc = (nk + KB - 1) / KB;
  const int bx = blockIdx.x, by = blockIdx.y;
  const int f = blockIdx.z / nkc, kc = blockIdx.z - f * nkc;
  int kk[KPT];
  float kt[KPT];
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int k = kc * KB + j * NT + tid;
    kk[j] = k < nk ? k : nk - 1;
    kt[j] = v.kturn[kk[j]];
  }
  const bool rot = !v.no_comp;
  const float W = (float)v.nu_w, inv2s2 = 0.5f / v.nu_s2;
  const int blk = (f * v.sp_nby + by) * v.sp_nbx + bx;
  const int e0 = v.sp_off[blk], e1 = v.sp_off[blk + 1];
  // accumulators: re / im parts of the cell pairs (2i, 2i+1), cell = cy*BX + cx
  float2 are[KPT][SP_CELLS / 2], aim[KPT][SP_CELLS / 2];
#pragma unroll
  for (int j = 0; j < KPT; ++j)
#pragma unroll
    for (int i = 0; i < SP_CELLS / 2; ++i) are[j][i] = aim[j][i] = make_float2(0.f, 0.f);
  for (int c0 = e0; c0 < e1; c0 += CH) {
    const int n = e1 - c0 < CH ? e1 - c0 : CH;
    __syncthreads();   // the previous round's weights are consumed
    {
      const int e = tid / SAR_SP_BY, cy = tid - e * SAR_SP_BY;
      if (e < n) {
        const SarSpreadEntry E = v.sp_ent[c0 + e];
        if (cy == 0) ent[e] = make_float4(__int_as_float(E.row), E.du, E.dv, E.beta);
        const float dy = (float)cy - E.dv;
        const float wy = fabsf(dy) <= W ? __expf(-dy * dy * inv2s2) : 0.f;
        float wr[SAR_SP_BX];
#pragma unroll
        for (int cx = 0; cx < SAR_SP_BX; ++cx) {
          const float dx = (float)cx - E.du;
          wr[cx] = fabsf(dx) <= W ? wy * __expf(-dx * dx * inv2s2) : 0.f;
        }
        float4 *dstw = reinterpret_cast<float4 *>(&wt[e][cy * SAR_SP_BX]);
#pragma unroll
        for (int q = 0; q < SAR_SP_BX / 4; ++q) dstw[q] = make_float4(wr[4 * q], wr[4 * q + 1], wr[4 * q + 2], wr[4 * q + 3]);
      }
    }
    __syncthreads();
    for (int e = 0; e < n; e += U) {
      float2 val[U][KPT];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int row = e + u < n ? __float_as_int(ent[e + u].x) : 0;
#pragma unroll
        for (int j = 0; j < KPT; ++j)
          val[u][j] = e + u < n ? __ldg(s + (size_t)row * nk + kk[j]) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (e + u < n) {
          float2 xr[KPT], xi[KPT];
#pragma unroll
          for (int j = 0; j < KPT; ++j) {
            float2 x = val[u][j];
            if (rot) {
              float turns = ent[e + u].w * kt[j];
              turns -= (turns + 12582912.f) - 12582912.f;   // round to nearest on the FMA pipe
              float sn, cs;
              __sincosf(turns * 6.28318530717958647692f, &sn, &cs);
              x = cmul(x, make_float2(cs, sn));
            }
            xr[j] = make_float2(x.x, x.x);
            xi[j] = make_float2(x.y, x.y);
          }
          const float4 *w4 = reinterpret_cast<const float4 *>(wt[e + u]);
#pragma unroll
          for (int i = 0; i < SP_CELLS / 4; ++i) {
            const float4 w = w4[i];
#pragma unroll
            for (int j = 0; j < KPT; ++j) {
              are[j][2 * i] = __ffma2_rn(xr[j], make_float2(w.x, w.y), are[j][2 * i]);
              are[j][2 * i + 1] = __ffma2_rn(xr[j], make_float2(w.z, w.w), are[j][2 * i + 1]);
              aim[j][2 * i] = __ffma2_rn(xi[j], make_float2(w.x, w.y), aim[j][2 * i]);
              aim[j][2 * i + 1] = __ffma2_rn(xi[j], make_float2(w.z, w.w), aim[j][2 * i + 1]);
            }
          }
        }
      }
    }
  }
  const int RX = 2 * v.nx, RY = 2 * v.ny;
  float2 *dst = v.wh + ((size_t)(f * RY + by * SAR_SP_BY) * RX + bx * SAR_SP_BX) * (size_t)nk;
#pragma unroll
  for (int j = 0; j < KPT; ++j) {
    const int k = kc * KB + j * NT + tid;
    if (k >= nk) continue;
#pragma unroll
    for (int i = 0; i < SP_CELLS / 2; ++i) {
      const int c = 2 * i, cy = c / SAR_SP_BX, cx = c - cy * SAR_SP_BX;
      float2 *d = dst + ((size_t)cy * RX + cx) * nk + k;
      __stcs(d, make_float2(are[j][i].x, aim[j][i].x));
      __stcs(d + nk, make_float2(are[j][i].y, aim[j][i].y));
    }
  }
}

// K2n: fine y-FFT of the x-transformed fine grid at the kept x frequencies,
// crop to |b_s| < ny/2, deconvolve by 1/(Phi_x Phi_y): W0.
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
  const int RX = 2 * nx;
  const int as = a < nx / 2 ? a : a - nx;
  const int af = as < 0 ? as + RX : as;
  const float dxa = __ldg(v.nu_decx + a);
  const float2 *src = v.wh + ((size_t)f * RY * RX + af) * (size_t)nk + kc * KC;
  const size_t row = (size_t)RX * nk;
  const size_t orow = (size_t)nx * nk;
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
          const float d = __ldg(v.nu_decy + b) * dxa;
          dst[(size_t)b * orow + c] = make_float2(x.x * d, x.y * d);
        }
      });
}

cudaError_t launch_k2n(const SarDeviceView &v, cudaStream_t s) {
  const int nchunk = (v.nk + KC - 1) / KC;
  dim3 grid(nchunk, v.nx, v.F);
  switch (2 * v.ny) {
#define X(N)                                                                                         \
  case N: {                                                                                          \
    const size_t smem = (size_t)N * KC * sizeof(float2);                                             \
    cudaError_t e = cudaFuncSetAttribute(k2n_yfft_crop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                  \
    k2n_yfft_crop<N><<<grid, sarfft2::nt_fft<N, KC>(), smem, s>>>(v);                          \
    return cudaGetLastError();                                                                       \
  }
    X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)
#undef X
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_k1s(const SarDeviceView &v, const float2 *data, cudaStream_t s) {
  // one wavenumber per thread, up to 256 per CTA
  const int kb = v.nk <= 64 ? 64 : (v.nk <= 128 ? 128 : 256);
  const int nkc = (v.nk + kb - 1) / kb;
  dim3 grid(v.sp_nbx, v.sp_nby, v.F * nkc);
  if (kb == 64) k1s_spread<64, 1><<<grid, 64, 0, s>>>(v, data);
  else if (kb == 128) k1s_spread<128, 1><<<grid, 128, 0, s>>>(v, data);
  else k1s_spread<256, 1><<<grid, 256, 0, s>>>(v, data);
  return cudaGetLastError();
}

}  // namespace

// SAR_GRID_NUFFT: part 1 = K1s spread; part 2 = fine x-FFT in place (the K2
// kernel on the fine grid viewed as [F*2ny][2nx][1][nk]) -> K2n (fine y-FFT,
// crop, 1/Phi).
cudaError_t launch_nufft(const SarDeviceView &v, const float2 *data, cudaStream_t s, const CUtensorMap *tm_fine,
                         int num_sms, int part) {
  if (part == 1) return launch_k1s(v, data, s);
  cudaError_t e = launch_mid<-1>(v.wh, v.tw_f, v.F * 2 * v.ny, 2 * v.nx, 1, v.nk, s, tm_fine, num_sms);
  if (e != cudaSuccess) return e;
  return launch_k2n(v, s);
}

}  // namespace sark
