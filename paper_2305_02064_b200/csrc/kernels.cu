// kernels.cu -- the five sm_100a kernels of the reconstruction path and their
// launchers.  Citation keys: P:n = PAPER.md line n; readings R1..R17 are in
// DESIGN.md section 3.
//
//   K1  k1_correct_xfft   per (frame, virtual row vy, 16-wide k chunk):
//                          gather every (tx,rx,pose) sample that lands on the
//                          row, rotate it by exp(+j k beta) (Eqs. (11)-(12),
//                          P:183-193), sum (reading R6), then FFT the row
//                          along x in shared memory.          raw -> W0
//   K2  k_fft_mid<-1>      FFT along y for (frame, kx, k chunk)   W0 -> W0
//   K3  k3_filter_stolt    per 8 (kx,ky) columns: filter k_z e^{+j k_z R_ref}/P
//                          on the source grid (readings R2-R4), linear
//                          Stolt pull onto the k_z grid (R5, R9),
//                          inverse FFT along z.               W0 -> W1
//   K4a k_fft_mid<+1>      inverse FFT along y                   W1 -> W1
//   K4b k4_xifft_mag       inverse FFT along x, |.|/(nx ny nz), integer rolls
//                          (R8, R11), transposed store to [f][z][y][x].  W1 -> image
//
// All transforms are the shared-memory Stockham FFT of fft_tile.cuh.  The
// path is HBM-bound: every kernel streams its input
// once with coalesced 128-byte row segments and keeps the transform on chip.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "fft_tile.cuh"
#include "plan_internal.h"

using sarfft::cadd;
using sarfft::cmul;

namespace {

constexpr int KC = 16;  // k (or z) chunk: 16 complex64 = one 128-byte line
constexpr double TWO_PI = 6.283185307179586476925286766559;
constexpr double BAND_EPS = 1e-9;  // reading R9

constexpr int nt_for(int n) { return n <= 32 ? 32 : (n < 512 ? n : 512); }

// ---------------------------------------------------------------- K1 ------
// One CTA = (k chunk, virtual row vy, frame f).  Thread item e covers
// (vx, kk) = (item / 16, item % 16).  For pair (t,r) the pose row feeding vy
// is iy = (vy - j^y_tr) mod ny (reading R6); it contributes iff iy < npy and
// ix = (vx - j^x_tr) mod nx < npx.  Rotation phase in turns:
// k_i beta / (2 pi) = kturn_i * (apose_p + bpair_tr), reduced to [-1/2, 1/2]
// before the SFU sincos (|k beta| reaches tens of radians).
template <int NX, bool DO_FFT>
__global__ void __launch_bounds__(nt_for(NX))
    k1_correct_xfft(const SarDeviceView v, const float2 *__restrict__ s) {
  constexpr int NT = nt_for(NX);
  constexpr int ITEMS = NX * KC;
  constexpr int E = (ITEMS + NT - 1) / NT;
  extern __shared__ float2 tile[];  // [NX][16]
  const int tid = threadIdx.x;
  const int kbase = blockIdx.x * KC;
  const int vy = blockIdx.y;
  const int f = blockIdx.z;

  float2 acc[E];
  float kt[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    acc[e] = make_float2(0.f, 0.f);
    const int k = kbase + ((tid + e * NT) & (KC - 1));
    kt[e] = k < v.nk ? __ldg(v.kturn + k) : 0.f;
  }

  for (int pr = 0; pr < v.npair; ++pr) {
    int iy = vy - v.jy[pr];
    if (iy < 0) iy += v.ny;
    if (iy >= v.npy) continue;  // uniform over the CTA
    const int t = pr / v.nr, r = pr - t * v.nr;
    const size_t rowbase = ((size_t)(f * v.nt + t) * v.nr + r) * (size_t)v.P + (size_t)iy * v.npx;
    const float2 *srow = s + rowbase * (size_t)v.nk;
    const float *ap = v.apose + (size_t)f * v.P + (size_t)iy * v.npx;
    const float bp = v.bpair[f * v.npair + pr];
    const int jx = v.jx[pr];
    // issue every load of this pair before consuming any (memory-level
    // parallelism: E independent 8-byte loads per thread in flight)
    float2 val[E];
    float bet[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int item = tid + e * NT;
      const int kk = item & (KC - 1);
      const int vx = item >> 4;
      int ix = vx - jx;
      if (ix < 0) ix += NX;
      const bool ok = (ITEMS % NT == 0 || item < ITEMS) && ix < v.npx && kbase + kk < v.nk;
      val[e] = ok ? __ldcs(srow + (size_t)ix * v.nk + (kbase + kk)) : make_float2(0.f, 0.f);
      bet[e] = ok ? __ldg(ap + ix) : 0.f;
    }
    if (v.no_comp) {
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = cadd(acc[e], val[e]);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        float turns = (bet[e] + bp) * kt[e];
        turns -= rintf(turns);
        float sn, cs;
        __sincosf(turns * 6.28318530717958647692f, &sn, &cs);
        acc[e] = cadd(acc[e], cmul(val[e], make_float2(cs, sn)));
      }
    }
  }

#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT == 0 || item < ITEMS) tile[item] = acc[e];  // tile[vx*16 + kk]
  }
  __syncthreads();
  if constexpr (DO_FFT) sarfft::tile_fft<NX, KC, KC, NT, -1>(tile, v.tw_x, tid);

  float2 *out = v.w0 + ((size_t)(f * v.ny + vy) * NX) * (size_t)v.nk;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int kk = item & (KC - 1), vx = item >> 4;
    const int k = kbase + kk;
    if (k < v.nk) out[(size_t)vx * v.nk + k] = tile[item];
  }
}

// ------------------------------------------------------------ K2 / K4a ----
// FFT along the middle (y) axis of a [F][N][nx][inner] complex volume for one
// (chunk of 16 along `inner`, column a, frame f).
template <int N, int DIR>
__global__ void __launch_bounds__(nt_for(N))
    k_fft_mid(float2 *__restrict__ data, const float2 *__restrict__ tw, int nx, int inner) {
  constexpr int NT = nt_for(N);
  constexpr int ITEMS = N * KC;
  constexpr int E = (ITEMS + NT - 1) / NT;
  extern __shared__ float2 tile[];  // [N][16]
  const int tid = threadIdx.x;
  const int cbase = blockIdx.x * KC;
  const int a = blockIdx.y;
  const int f = blockIdx.z;
  float2 *base = data + ((size_t)f * N * nx + a) * (size_t)inner;
  const size_t row = (size_t)nx * inner;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int cc = item & (KC - 1), b = item >> 4;
    const int c = cbase + cc;
    tile[item] = c < inner ? base[b * row + c] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  sarfft::tile_fft<N, KC, KC, NT, DIR>(tile, tw, tid);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int cc = item & (KC - 1), b = item >> 4;
    const int c = cbase + cc;
    if (c < inner) base[b * row + c] = tile[item];
  }
}

// ---------------------------------------------------------------- K3 ------
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
  const double fl = floor(u);
  const bool near = u < delta || u > (double)(nk - 1) - delta || (u - fl) < delta || (u - fl) > 1.0 - delta;
  if (near) return stolt_pull_exact(kzj, kr2, k0, dk, nk, i0, tau);
  *i0 = (int)fl;
  *tau = u - fl;
  return true;
}

__device__ __forceinline__ double kr2_of(const SarDeviceView &v, int a, int b) {
  const double kx = v.kx[a], ky = v.ky[b];
  return __dadd_rn(__dmul_rn(kx, kx), __dmul_rn(ky, ky));
}

constexpr int K3_CC = 8;              // columns per CTA
constexpr int K3_LD = K3_CC + 1;      // padded row stride of the [n][CC] tiles
constexpr int K3_NT = 256;

template <int NZ, bool DO_IFFT>
__global__ void __launch_bounds__(K3_NT) k3_filter_stolt(const SarDeviceView v) {
  extern __shared__ float2 sm[];
  float2 *fin = sm;                          // [nk][LD]  filtered source spectrum
  float2 *fout = sm + (size_t)v.nk * K3_LD;  // [NZ][LD]  Stolt output
  double *kr2s = reinterpret_cast<double *>(fout + (size_t)NZ * K3_LD);  // [CC]
  const int tid = threadIdx.x;
  const int ncol = v.nx * v.ny;
  const int col0 = blockIdx.x * K3_CC;
  const int f = blockIdx.y;
  const int nk = v.nk;
  if (tid < K3_CC) {
    const int col = min(col0 + tid, ncol - 1);
    kr2s[tid] = kr2_of(v, col % v.nx, col / v.nx);
  }
  __syncthreads();
  const double rref = v.rref[f];
  const float2 *src = v.w0 + ((size_t)f * ncol + col0) * (size_t)nk;
  const int ncc = min(K3_CC, ncol - col0);
  // 1. load + filter H = k_z exp(+j k_z R_ref) / P(f) on the source grid
  for (int c = 0; c < K3_CC; ++c) {
    const double kr2 = kr2s[c];
    for (int i = tid; i < nk; i += K3_NT) {
      float2 val = make_float2(0.f, 0.f);
      if (c < ncc) {
        const double ki = v.k[i];
        const double q = 4.0 * ki * ki - kr2;
        if (q > 0.0) {
          const double kz = fast_dsqrt(q);
          double turns = kz * rref * (1.0 / TWO_PI);
          turns -= rint(turns);
          float sn, cs;
          __sincosf((float)turns * 6.28318530717958647692f, &sn, &cs);
          const float kzf = (float)kz;
          float2 h = make_float2(kzf * cs, kzf * sn);
          if (v.pinv) h = cmul(h, v.pinv[i]);
          val = cmul(__ldcs(src + (size_t)c * nk + i), h);
        }
      }
      fin[i * K3_LD + c] = val;
    }
  }
  __syncthreads();
  // 2. Stolt pull onto the uniform k_z grid
  for (int idx = tid; idx < K3_CC * NZ; idx += K3_NT) {
    const int c = idx % K3_CC, j = idx / K3_CC;
    int i0;
    double tau;
    float2 o = make_float2(0.f, 0.f);
    if (stolt_pull(v.kz[j], kr2s[c], v.k0, v.inv_dk, v.dk, nk, v.stolt_delta, &i0, &tau)) {
      const float t = (float)tau;
      const float2 lo = fin[i0 * K3_LD + c], hi = fin[(i0 + 1) * K3_LD + c];
      o = make_float2(fmaf(t, hi.x - lo.x, lo.x), fmaf(t, hi.y - lo.y, lo.y));
    }
    fout[j * K3_LD + c] = o;
  }
  __syncthreads();
  // 3. inverse FFT along z
  if constexpr (DO_IFFT) sarfft::tile_fft<NZ, K3_CC, K3_LD, K3_NT, +1>(fout, v.tw_z, tid);
  // 4. store column-contiguous [col][z]
  float2 *dst = v.w1 + ((size_t)f * ncol + col0) * (size_t)NZ;
  for (int idx = tid; idx < ncc * NZ; idx += K3_NT) {
    const int c = idx / NZ, z = idx - c * NZ;
    dst[idx] = fout[z * K3_LD + c];
  }
}

__global__ void k_stolt_index(const SarDeviceView v, const int32_t *__restrict__ cols, int n,
                              int32_t *__restrict__ i0_out, float *__restrict__ tau_out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n * v.nz) return;
  const int c = (int)(idx / v.nz), j = (int)(idx - (long long)c * v.nz);
  const int a = cols[2 * c], b = cols[2 * c + 1];
  int i0;
  double tau;
  if (a >= 0 && a < v.nx && b >= 0 && b < v.ny &&
      stolt_pull(v.kz[j], kr2_of(v, a, b), v.k0, v.inv_dk, v.dk, v.nk, v.stolt_delta, &i0, &tau)) {
    i0_out[idx] = i0;
    tau_out[idx] = (float)tau;
  } else {
    i0_out[idx] = -1;
    tau_out[idx] = 0.f;
  }
}

// --------------------------------------------------------------- K4b ------
// One CTA = (z chunk, image row y (pre-roll), frame).  Tile [NX][17]: the odd
// stride makes both the FFT passes and the transposed read conflict-free.
template <int NX, bool CPLX>
__global__ void __launch_bounds__(nt_for(NX))
    k4_xifft_mag(const SarDeviceView v, void *__restrict__ img) {
  constexpr int NT = nt_for(NX);
  constexpr int LD = KC + 1;
  constexpr int ITEMS = NX * KC;
  constexpr int E = (ITEMS + NT - 1) / NT;
  extern __shared__ float2 tile[];  // [NX][LD]
  const int tid = threadIdx.x;
  const int zbase = blockIdx.x * KC;
  const int y = blockIdx.y;
  const int f = blockIdx.z;
  const int nz = v.nz;
  const float2 *src = v.w1 + ((size_t)(f * v.ny + y) * NX) * (size_t)nz;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int zz = item & (KC - 1), a = item >> 4;
    const int z = zbase + zz;
    tile[a * LD + zz] = z < nz ? src[(size_t)a * nz + z] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  sarfft::tile_fft<NX, KC, LD, NT, +1>(tile, v.tw_x, tid);
  int iy = y - v.roll_y % v.ny;
  if (iy < 0) iy += v.ny;
  if (iy >= v.ny) iy -= v.ny;
  const int rx = ((v.roll_x % NX) + NX) % NX;
  const float sc = v.img_scale;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int zz = item / NX, ix = item - zz * NX;
    const int z = zbase + zz;
    if (z >= nz) continue;
    int m = z + nz / 2;
    if (m >= nz) m -= nz;
    const int xs = (ix + rx) & (NX - 1);
    const float2 o = tile[xs * LD + zz];
    const size_t off = ((size_t)(f * nz + m) * v.ny + iy) * NX + ix;
    if constexpr (CPLX) {
      reinterpret_cast<float2 *>(img)[off] = make_float2(o.x * sc, o.y * sc);
    } else {
      reinterpret_cast<float *>(img)[off] = sqrtf(fmaf(o.x, o.x, o.y * o.y)) * sc;
    }
  }
}

// ------------------------------------------------------------ dispatch ----
#define SAR_SIZES(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)

template <typename K>
cudaError_t launch(K kernel, dim3 grid, int nt, size_t smem, cudaStream_t s, const SarDeviceView &v,
                   const float2 *arg) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, nt, smem, s>>>(v, arg);
  return cudaGetLastError();
}

cudaError_t launch_k1(const SarDeviceView &v, const float2 *data, bool fft, cudaStream_t s) {
  dim3 grid((v.nk + KC - 1) / KC, v.ny, v.F);
  const size_t smem = (size_t)v.nx * KC * sizeof(float2);
  switch (v.nx) {
#define X(N)                                                                                   \
  case N:                                                                                      \
    return fft ? launch(k1_correct_xfft<N, true>, grid, nt_for(N), smem, s, v, data)          \
               : launch(k1_correct_xfft<N, false>, grid, nt_for(N), smem, s, v, data);
    SAR_SIZES(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

template <int DIR>
cudaError_t launch_mid(float2 *data, const float2 *tw, int F, int ny, int nx, int inner, cudaStream_t s) {
  dim3 grid((inner + KC - 1) / KC, nx, F);
  const size_t smem = (size_t)ny * KC * sizeof(float2);
  switch (ny) {
#define X(N)                                                                                       \
  case N: {                                                                                        \
    auto kern = k_fft_mid<N, DIR>;                                                                 \
    if (smem > 48 * 1024) {                                                                        \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (e != cudaSuccess) return e;                                                              \
    }                                                                                              \
    kern<<<grid, nt_for(N), smem, s>>>(data, tw, nx, inner);                                       \
    return cudaGetLastError();                                                                     \
  }
    SAR_SIZES(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

template <typename K>
cudaError_t launch_v(K kernel, dim3 grid, int nt, size_t smem, cudaStream_t s, const SarDeviceView &v) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, nt, smem, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_k3(const SarDeviceView &v, bool ifft, cudaStream_t s) {
  const int ncol = v.nx * v.ny;
  dim3 grid((ncol + K3_CC - 1) / K3_CC, v.F);
  const size_t smem = (size_t)(v.nk + v.nz) * K3_LD * sizeof(float2) + K3_CC * sizeof(double);
  switch (v.nz) {
#define X(N)                                                                           \
  case N:                                                                              \
    return ifft ? launch_v(k3_filter_stolt<N, true>, grid, K3_NT, smem, s, v)          \
                : launch_v(k3_filter_stolt<N, false>, grid, K3_NT, smem, s, v);
    SAR_SIZES(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

template <typename K>
cudaError_t launch_img(K kernel, dim3 grid, int nt, size_t smem, cudaStream_t s, const SarDeviceView &v,
                       void *img) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, nt, smem, s>>>(v, img);
  return cudaGetLastError();
}

cudaError_t launch_k4b(const SarDeviceView &v, void *img, bool cplx, cudaStream_t s) {
  dim3 grid((v.nz + KC - 1) / KC, v.ny, v.F);
  const size_t smem = (size_t)v.nx * (KC + 1) * sizeof(float2);
  switch (v.nx) {
#define X(N)                                                                             \
  case N:                                                                                \
    return cplx ? launch_img(k4_xifft_mag<N, true>, grid, nt_for(N), smem, s, v, img)    \
                : launch_img(k4_xifft_mag<N, false>, grid, nt_for(N), smem, s, v, img);
    SAR_SIZES(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// Enqueue the path.  stop_stage: 0 = full; 1 = K1 without the x-FFT; 2 = K1+K2;
// 3 = K1+K2+K3 without the z-IFFT.  ev (optional, 6 events) brackets the kernels.
int sar_launch_pipeline(sar_plan *p, const void *d_data, void *d_image, cudaStream_t s, int stop_stage,
                        int complex_out, cudaEvent_t *ev) {
  const SarDeviceView &v = p->v;
  const float2 *data = reinterpret_cast<const float2 *>(d_data);
  cudaError_t e = cudaSuccess;
#define SAR_CHECK(call)                                                       \
  do {                                                                        \
    e = (call);                                                               \
    if (e != cudaSuccess) {                                                   \
      sar_set_error(std::string("CUDA: ") + cudaGetErrorString(e) + " in " #call); \
      return SAR_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)
  if (ev) SAR_CHECK(cudaEventRecord(ev[0], s));
  SAR_CHECK(launch_k1(v, data, stop_stage != 1, s));
  if (ev) SAR_CHECK(cudaEventRecord(ev[1], s));
  if (stop_stage == 1) return SAR_OK;
  SAR_CHECK(launch_mid<-1>(v.w0, v.tw_y, v.F, v.ny, v.nx, v.nk, s));
  if (ev) SAR_CHECK(cudaEventRecord(ev[2], s));
  if (stop_stage == 2) return SAR_OK;
  SAR_CHECK(launch_k3(v, stop_stage != 3, s));
  if (ev) SAR_CHECK(cudaEventRecord(ev[3], s));
  if (stop_stage == 3) return SAR_OK;
  SAR_CHECK(launch_mid<+1>(v.w1, v.tw_y, v.F, v.ny, v.nx, v.nz, s));
  if (ev) SAR_CHECK(cudaEventRecord(ev[4], s));
  SAR_CHECK(launch_k4b(v, d_image, complex_out != 0, s));
  if (ev) SAR_CHECK(cudaEventRecord(ev[5], s));
  return SAR_OK;
}

int sar_launch_stolt_index(sar_plan *p, const int32_t *d_cols, int n, int32_t *d_i0, float *d_tau,
                           cudaStream_t s) {
  const long long total = (long long)n * p->v.nz;
  if (total == 0) return SAR_OK;
  const int nt = 256;
  const long long nb = (total + nt - 1) / nt;
  k_stolt_index<<<(unsigned)nb, nt, 0, s>>>(p->v, d_cols, n, d_i0, d_tau);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    sar_set_error(std::string("CUDA: ") + cudaGetErrorString(e));
    return SAR_ERR_CUDA;
  }
  return SAR_OK;
}
