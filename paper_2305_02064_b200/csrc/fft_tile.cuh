// fft_tile.cuh -- batched radix-8/4/2 Stockham FFTs over a shared-memory tile.
//
// Used by every transform of the path: FT_2D and IFT_3D of Eq. (14).
// A tile holds C independent columns of length N:  x[n*LD + c]  (n in [0,N),
// c in [0,C)), i.e. the batch index is the fastest one, so a warp touches
// consecutive complex words and every global load/store of a tile row is a
// coalesced 8*C-byte segment.  The transform is unnormalised; DIR = -1 is the
// forward e^{-2 pi i nk/N} (numpy convention, reading R2), DIR = +1 the inverse.
//
// Stockham autosort pass with radix R at span P (P = product of the radices
// already applied):  for butterfly i in [0, N/R):  k = i mod P,
//   u_r = x[i + r N/R] * W_{P R}^{r k}   (r = 0..R-1)
//   y[(i - k) R + k + r P] = DFT_R(u)_r
// which leaves the result in natural order after the last pass.  Each pass
// keeps its inputs in registers between two __syncthreads(), so it runs in
// place.  Twiddles come from a table tw[m] = exp(-2 pi i m / N) (fp64 on the
// host, rounded once to fp32); the inverse uses the conjugate.
#pragma once
#include <cuda_runtime.h>

namespace sarfft {

// Complex arithmetic on the sm_100 paired-fp32 pipe (FADD2 / FMUL2 / FFMA2):
// one instruction per complex add, two per complex multiply.
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(-a.y, a.y), make_float2(b.y, b.x)));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
// multiply by -i (DIR = -1) or +i (DIR = +1)
template <int DIR>
__device__ __forceinline__ float2 mul_mi(float2 a) {
  return DIR < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}

template <int DIR>
__device__ __forceinline__ void dft2(float2 *v) {
  float2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <int DIR>
__device__ __forceinline__ void dft4(float2 *v) {
  float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
  float2 t2 = cadd(v[1], v[3]), t3 = mul_mi<DIR>(csub(v[1], v[3]));
  v[0] = cadd(t0, t2);
  v[2] = csub(t0, t2);
  v[1] = cadd(t1, t3);
  v[3] = csub(t1, t3);
}

// radix-8 = one radix-2 stage (pairs r, r+4, twiddles W8^r) + two radix-4 DFTs
template <int DIR>
__device__ __forceinline__ void dft8(float2 *v) {
  const float h = 0.70710678118654752440f;
  float2 b[4], c[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    b[r] = cadd(v[r], v[r + 4]);
    c[r] = csub(v[r], v[r + 4]);
  }
  // c_r *= W8^{r} with W8 = exp(DIR * 2 pi i / 8)
  const float2 hh = make_float2(h, h);
  c[1] = DIR < 0 ? __fmul2_rn(hh, __fadd2_rn(c[1], make_float2(c[1].y, -c[1].x)))
                 : __fmul2_rn(hh, __fadd2_rn(c[1], make_float2(-c[1].y, c[1].x)));
  c[2] = mul_mi<DIR>(c[2]);
  c[3] = DIR < 0 ? __fmul2_rn(hh, __fadd2_rn(make_float2(c[3].y, -c[3].x), make_float2(-c[3].x, -c[3].y)))
                 : __fmul2_rn(hh, __fadd2_rn(make_float2(-c[3].y, c[3].x), make_float2(-c[3].x, -c[3].y)));
  dft4<DIR>(b);
  dft4<DIR>(c);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    v[2 * m] = b[m];
    v[2 * m + 1] = c[m];
  }
}

template <int R, int DIR>
__device__ __forceinline__ void dft(float2 *v) {
  if constexpr (R == 8) dft8<DIR>(v);
  else if constexpr (R == 4) dft4<DIR>(v);
  else dft2<DIR>(v);
}

// Block barrier: BARID 0 = __syncthreads(); otherwise a named barrier over the
// NT threads that run the transform (warp-specialised kernels keep their
// producer warp out of it).
template <int BARID, int NT>
__device__ __forceinline__ void tile_sync() {
  if constexpr (BARID == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"n"(BARID), "n"(NT) : "memory");
  }
}

template <int REM>
struct radix_for {
  static constexpr int value = (REM % 8 == 0 && REM != 16) ? 8 : (REM % 4 == 0 ? 4 : 2);
};

// One Stockham pass.  NT threads, tid in [0, NT).
template <int N, int C, int LD, int NT, int DIR, int R, int P, int BARID>
__device__ __forceinline__ void stockham_pass(float2 *x, const float2 *__restrict__ tw, int tid) {
  constexpr int NR = N / R;
  constexpr int ITEMS = C * NR;              // butterflies in the tile
  constexpr int IT = (ITEMS + NT - 1) / NT;  // per thread
  float2 v[IT][R];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int item = tid + it * NT;
    if (ITEMS % NT == 0 || item < ITEMS) {
      const int c = item % C, i = item / C;
#pragma unroll
      for (int r = 0; r < R; ++r) v[it][r] = x[(i + r * NR) * LD + c];
    }
  }
  tile_sync<BARID, NT>();
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int item = tid + it * NT;
    if (ITEMS % NT == 0 || item < ITEMS) {
      const int c = item % C, i = item / C;
      const int k = i % P;
      if constexpr (P > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const int idx = (r * k * (N / (P * R))) % N;
          float2 w = tw[idx];
          if (DIR > 0) w.y = -w.y;
          v[it][r] = cmul(v[it][r], w);
        }
      }
      dft<R, DIR>(v[it]);
      const int j = (i - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) x[(j + r * P) * LD + c] = v[it][r];
    }
  }
  tile_sync<BARID, NT>();
}

template <int N, int C, int LD, int NT, int DIR, int P, int BARID>
__device__ __forceinline__ void fft_passes(float2 *x, const float2 *__restrict__ tw, int tid) {
  if constexpr (P < N) {
    constexpr int R = radix_for<N / P>::value;
    stockham_pass<N, C, LD, NT, DIR, R, P, BARID>(x, tw, tid);
    fft_passes<N, C, LD, NT, DIR, P * R, BARID>(x, tw, tid);
  }
}

// In-place FFT of the C columns of tile x (length N, row stride LD).  Must be
// called by all NT threads (tid in [0, NT)); ends with a barrier.
template <int N, int C, int LD, int NT, int DIR, int BARID = 0>
__device__ __forceinline__ void tile_fft(float2 *x, const float2 *__restrict__ tw, int tid) {
  static_assert((N & (N - 1)) == 0 && N >= 2, "power-of-two length");
  fft_passes<N, C, LD, NT, DIR, 1, BARID>(x, tw, tid);
}

}  // namespace sarfft
