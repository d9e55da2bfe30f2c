// common.cuh -- device helpers, constants and launcher declarations shared by
// the kernel translation units (k1.cu, fft_mid.cu, k3.cu, k4.cu,
// nufft.cu) and the pipeline (pipeline.cu).  Citation keys: P:n = PAPER.md
// line n; readings R1..R19 are in DESIGN.md section 3.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_reg.cuh"
#include "fft_tile.cuh"
#include "plan_internal.h"
#include "tma.cuh"

namespace sark {

using sarfft::cadd;
using sarfft::cmul;

constexpr int KC = 16;  // k (or z) chunk: 16 complex64 = one 128-byte line

// SAR_CHECKED builds (`build.py --variant=checked -DSAR_CHECKED`, testing only;
// compute-sanitizer is closed on the GPU pool): every global store / bulk copy
// of the path and the shared-memory indices of the warp-specialised kernels
// are checked against their buffer and trap with a message when outside
#ifdef SAR_CHECKED
#define SAR_ASSERT(c)                                                                        \
  do {                                                                                       \
    if (!(c)) {                                                                              \
      printf("SAR_CHECKED %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x,   \
             threadIdx.x, #c);                                                               \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)
#else
#define SAR_ASSERT(c) ((void)0)
#endif
// p inside [base, base + n elements)
#define SAR_IN(p, base, n) SAR_ASSERT((p) >= (base) && (p) < (base) + (n))
constexpr double TWO_PI = 6.283185307179586476925286766559;
constexpr double BAND_EPS = 1e-9;  // reading R9

constexpr int nt_for(int n) { return n <= 32 ? 32 : (n < 512 ? n : 512); }
// resident CTAs requested per SM: 1024 threads' worth (caps registers at 64 per
// thread) except for the 1024-point tiles, whose 32 elements per thread need more
constexpr int minb_for(int n) { return n >= 1024 ? 1 : 1024 / nt_for(n); }

#ifndef K1_STAGES_
#define K1_STAGES_ 4
#endif
#ifndef K1_BOX_BYTES_
#define K1_BOX_BYTES_ 32768
#endif
constexpr int K1_STAGES = K1_STAGES_;        // TMA ring stages of K1
constexpr int K1_BOX_BYTES = K1_BOX_BYTES_;  // raw-sample bytes per TMA box
constexpr int K1_NT = 512;   // consumer threads (+1 producer warp)
#ifndef K1_KT_
#define K1_KT_ 4
#endif
constexpr int K1_KT = K1_KT_;  // consecutive k per thread (one SFU sincos + step phasor per K1_KT samples)

constexpr int k1c_for(int nx) { return nx >= 256 ? 16 : 64; }

// Store of an intermediate volume (W0 / W1) that the next kernel reads:
// default write-back caching, so a frame wave's volumes can be served from
// L2 (plan.cpp: frame waves); SAR_STREAM_INTERMEDIATES selects the
// evict-first streaming store instead (A/B builds)
__device__ __forceinline__ void st_mid(float2 *p, float2 x) {
#ifdef SAR_STREAM_INTERMEDIATES
  __stcs(p, x);
#else
  *p = x;
#endif
}

// acc += a * b (complex), two paired-fp32 FMAs
__device__ __forceinline__ float2 cmac2(float2 acc, float2 a, float2 b) {
  acc = __ffma2_rn(make_float2(a.x, a.x), b, acc);
  return __ffma2_rn(make_float2(-a.y, a.y), make_float2(b.y, b.x), acc);
}
__device__ __forceinline__ float2 cmul2(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(-a.y, a.y), make_float2(b.y, b.x)));
}

// Stolt pull index (readings R4, R5, R9).  The decisions (in band? which
// interval?) must equal oracle.stolt_index_table bit for bit, which evaluates
// in fp64 without contraction
//   ks = kz*kz + kr2;  kk = 0.5*sqrt(ks);  u = (kk - k0)/dk.
// stolt_pull_exact does exactly that (IEEE sqrt/div intrinsics).  The fast
// path computes u with one fp32 rsqrt + one fp64 Newton step (relative error
// <= 1.5 e^2 ~ 1e-13 for the ~2^-22 rsqrt seed) and a multiplication by 1/dk;
// whenever that estimate lies within `delta` (100x its error bound, >= 1e-7,
// set by the plan) of a decision boundary -- a band edge or an integer -- the
// exact sequence decides, so the decisions are identical to the exact path
// everywhere and tau differs by far less than its fp32 rounding.
__device__ __forceinline__ bool stolt_pull_exact(double kzj, double kr2, double k0, double dk, int nk,
                                                 int *i0, double *tau) {
  if (!(kzj > 0.0)) return false;
  const double ks = __dadd_rn(__dmul_rn(kzj, kzj), kr2);
  const double kk = __dmul_rn(0.5, __dsqrt_rn(ks));
  const double u = __ddiv_rn(__dsub_rn(kk, k0), dk);
  const double hi = __dadd_rn((double)(nk - 1), BAND_EPS);
  if (!(u >= -BAND_EPS && u <= hi)) return false;
  const double uc = fmin(fmax(u, 0.0), (double)(nk - 1));
  int i = (int)floor(uc);
  if (i > nk - 2) i = nk - 2;
  *i0 = i;
  *tau = __dsub_rn(uc, (double)i);
  return true;
}

// sqrt(x) for x > 0 to ~1e-15 relative: fp32 rsqrt seed + one Newton step in fp64
__device__ __forceinline__ double fast_dsqrt(double x) {
  const double y = (double)rsqrtf((float)x);
  const double s0 = x * y;
  return fma(0.5 * y, fma(-s0, s0, x), s0);
}

__device__ __forceinline__ bool stolt_pull(double kzj, double kr2, double k0, double inv_dk, double dk, int nk,
                                           double delta, int *i0, double *tau) {
  if (!(kzj > 0.0)) return false;
  const double u = (0.5 * fast_dsqrt(fma(kzj, kzj, kr2)) - k0) * inv_dk;
  const double top = (double)(nk - 1);
  // clearly out of band (|u - u_exact| << delta and the edges sit within
  // BAND_EPS << delta of 0 and n_k-1)
  if (u < -delta || u > top + delta) return false;
  const double fl = floor(u);
  const bool near = u < delta || u > top - delta || (u - fl) < delta || (u - fl) > 1.0 - delta;
  if (near) return stolt_pull_exact(kzj, kr2, k0, dk, nk, i0, tau);
  *i0 = (int)fl;
  *tau = u - fl;
  return true;
}

__device__ __forceinline__ double kr2_of(const SarDeviceView &v, int a, int b) {
  const double kx = v.kx[a], ky = v.ky[b];
  return __dadd_rn(__dmul_rn(kx, kx), __dmul_rn(ky, ky));
}

// Filter value H(k_r, k_i) = k_z e^{+j k_z R_ref} / P(f_i) (0 when evanescent),
// readings R2-R4; rr = R_ref / (2 pi), phase reduced in turns.
__device__ __forceinline__ float2 filter_h(const SarDeviceView &v, double ki, double kr2, double rr, int i) {
  const double q = 4.0 * ki * ki - kr2;
  float2 hh = make_float2(0.f, 0.f);
  if (q > 0.0) {
    const double kz = fast_dsqrt(q);
    double turns = kz * rr;
    turns -= rint(turns);
    float sn, cs;
    __sincosf((float)turns * 6.28318530717958647692f, &sn, &cs);
    const float kzf = (float)kz;
    hh = make_float2(kzf * cs, kzf * sn);
    if (v.pinv) hh = cmul(hh, v.pinv[i]);
  }
  return hh;
}

// U independent evaluations per thread of the filter table [CL][nk] (ILP for
// the fp64 chains); idx = t0 + u*stride
template <int U, typename KR2, typename KS>
__device__ __forceinline__ void filter_table(const SarDeviceView &v, float2 *htab, int total, int nk, int t0,
                                             int stride, double rr, KR2 &&kr2_of_cl, KS &&ks) {
  for (int base = t0; base < total; base += U * stride) {
    float2 hv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = base + u * stride;
      hv[u] = make_float2(0.f, 0.f);
      if (idx < total) {
        const int cl = idx / nk, i = idx - cl * nk;
        hv[u] = filter_h(v, ks(i), kr2_of_cl(cl), rr, i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = base + u * stride;
      if (idx < total) htab[idx] = hv[u];
    }
  }
}

// K3 for the large grids: persistent, warp-specialised, ping-pong.  A
// producer warp decodes work items (CL mirror classes = up to 4*CL spectral
// columns that share k_r^2) into an S-stage ring and fills it with TMA bulk
// copies (one n_k-sample column each, mbarrier completion).  Two consumer
// groups of 256 threads take alternate items, so one group's fp64 filter /
// Stolt phases and barrier waits overlap the other group's FFT.  Per item:
// (1) filter table H(k_r, k_i) = k_z e^{+j k_z R_ref}/P once per class;
// (2) Stolt pull with the filter folded into the two interpolation weights,
// once per (class, j), applied to every member column (decisions bit-exact,
// readings R5, R9); the stage is then handed back; (3) inverse z-FFT (two-pass
// register FFT) whose pass 2 stores each column contiguously [col][z].
// The k, k_z and twiddle tables live in shared memory.
template <int CL>
struct K3Hdr {
  double rr;               // R_ref(f) / (2 pi), read by the producer
  int f, nused;
  int nmem[CL], mslot[CL][4];
  int jlo[CL], jhi[CL];   // in-band k_z bins of the class (superset, see stolt_range)
  int colof[4 * CL], clof[4 * CL];
  double kr2[CL];
};

// Superset [jlo, jhi] of the k_z bins j whose Stolt pull can be in band for
// k_r^2 = kr2 (readings R5, R9): u(j) is monotone in j, u = 0 at
// k_z = sqrt(4 k_0^2 - k_r^2) and u = n_k - 1 at sqrt(4 k_max^2 - k_r^2); the
// range is widened by 2 bins on each side (the estimate is good to ~1e-12
// bins), and to the whole axis when a band edge lies within 1e-3 bins of
// k_z = 0 (where du/dj -> 0 and the margin would not cover the 1e-9 band
// tolerance).  Bins outside the range are zero; inside, the bit-exact pull
// decides.
__device__ __forceinline__ void stolt_range(const SarDeviceView &v, double kr2, int *jlo, int *jhi) {
  const int nz = v.nz;
  const double kmax = v.k0 + (double)(v.nk - 1) * v.dk;
  const double qhi = 4.0 * kmax * kmax - kr2;
  if (!(qhi > 0.0)) {
    *jlo = 0;
    *jhi = -1;
    return;
  }
  const double qlo = 4.0 * v.k0 * v.k0 - kr2;
  const double kzhi = sqrt(qhi), kzlo = qlo > 0.0 ? sqrt(qlo) : 0.0;
  const double guard = 1e-3 * v.kz_step;
  if (kzlo < guard || kzhi < guard) {
    *jlo = 0;
    *jhi = nz - 1;
    return;
  }
  const double jl = (double)(nz - 1) - (v.kz_top - kzlo) / v.kz_step;
  const double jh = (double)(nz - 1) - (v.kz_top - kzhi) / v.kz_step;
  int lo = (int)fmax(floor(jl) - 2.0, 0.0);
  int hi = (int)fmin(ceil(jh) + 2.0, (double)(nz - 1));
  *jlo = lo;
  *jhi = hi < lo ? lo - 1 : hi;
}
// CTAs of `kern` resident per SM (cached); the persistent grids never exceed
// num_sms times it
int resident_ctas(const void *kern, int threads, size_t smem);

// launch through cudaLaunchKernelEx (no attributes: programmatic dependent
// launch between the five kernels was measured slower, 3.534 vs 3.504 ms on
// Large)
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = nullptr;
  cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

#define SAR_SIZES(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)

// ---- launchers (one translation unit each) ----
cudaError_t launch_k1(const SarDeviceView &v, const float2 *data, bool fft, cudaStream_t s,
                      const CUtensorMap *tm_s, const CUtensorMap *tm_ap, int br, bool regacc, int num_sms);
// Optional slab epilogue of the mid-axis FFT (slab stage 2, K4a): chunk c of
// column a goes to block h = c*16 / nzl (the packed send buffer or a peer's
// receive buffer) at [row][a][z - h nzl] with nzl z-slots per block.
struct MidSlabOut {
  char *d[SAR_MAX_SLAB];
  int nzl;   // 0: off (in place)
};
// liveb (or nullptr = every row): [nx] live-row bound of each column a, the
// rows |m_s| <= liveb[a].  Forward (K2): only live rows
// are stored.  Inverse (K4a): only live rows are read, the others are zero.
// tm_st (or nullptr): a [32 rows][16] box map over `data` for TMA stores of
// the transformed tiles (ny >= 256)
template <int DIR>
cudaError_t launch_mid(float2 *data, const float2 *tw, int F, int ny, int nx, int inner, cudaStream_t s,
                       const CUtensorMap *tm, int num_sms, const MidSlabOut *so = nullptr,
                       const int *liveb = nullptr, const CUtensorMap *tm_st = nullptr);
cudaError_t launch_k3(const SarDeviceView &v, bool ifft, cudaStream_t s, int num_sms);

cudaError_t launch_k3_plane(const SarDeviceView &v, cudaStream_t s);
cudaError_t launch_stolt_index(const SarDeviceView &v, const int32_t *cols, int n, int32_t *i0, float *tau,
                               cudaStream_t s);
cudaError_t launch_k4b(const SarDeviceView &v, void *img, bool cplx, cudaStream_t s, const CUtensorMap *tm,
                       int num_sms, bool slab4d = false);
cudaError_t launch_nufft(const SarDeviceView &v, const float2 *data, cudaStream_t s, const CUtensorMap *tm_fine,
                         int num_sms, int part);

}  // namespace sark
