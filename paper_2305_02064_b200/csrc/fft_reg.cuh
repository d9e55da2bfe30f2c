// fft_reg.cuh -- two-pass, register-resident batched FFTs for sm_100a.
//
// Used by every transform of the path: FT_2D and IFT_3D of Eq. (14).
// A batch of C independent columns of length N (power of two, 2..1024) is
// transformed in at most two Stockham passes N = R1 * R2 (R1, R2 <= 32):
//
//   pass 1 (radix R1, span 1):  for column c, butterfly i in [0, R2):
//       u_r = x[i + r R2]                       r = 0..R1-1
//       y[i R1 + p] = DFT_R1(u)_p               (shared-memory work tile)
//   pass 2 (radix R2, span R1): for column c, butterfly i in [0, R1):
//       u_r = y[i + r R1] * W_N^{r i}           r = 0..R2-1
//       X[i + p R1] = DFT_R2(u)_p
//
// which is the unnormalised DFT X[n] = sum_m x[m] exp(DIR 2 pi i m n / N)
// (DIR = -1 forward, numpy sign; DIR = +1 inverse; reading R2).  Each
// butterfly is an in-register radix-4/2 decimation-in-frequency DFT with
// compile-time twiddles (trivial ones cost nothing, the 1/8-turn ones two
// instructions), so the only shared-memory traffic is one store and one load
// per element between the passes plus one table load per element for the
// inter-pass twiddle (host fp64 table rounded once to fp32).
//
// The input of pass 1 and the output of pass 2 go through caller functors
// load(c, n) -> float2 and store(c, n, float2), so producers (a TMA stage, the
// Stolt interpolation) and consumers (global stores, the magnitude epilogue)
// fuse into the passes instead of round-tripping through shared memory.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

namespace sarfft2 {

// ---- compile-time helpers -------------------------------------------------
constexpr double kPi = 3.14159265358979323846264338327950288;
constexpr double sin_series(double x) {
  double term = x, sum = x;
  for (int n = 1; n < 40; ++n) {
    term *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
    sum += term;
  }
  return sum;
}
constexpr double cos_series(double x) {
  double term = 1.0, sum = 1.0;
  for (int n = 1; n < 40; ++n) {
    term *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
    sum += term;
  }
  return sum;
}
constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// W_L^M = exp(DIR 2 pi i M / L), angle reduced to [-pi, pi]
template <int M, int L, int DIR>
struct Tw {
  static constexpr int m = ((M % L) + L) % L;
  static constexpr double turns = (2 * m > L) ? (double)(m - L) / L : (double)m / L;
  static constexpr double ang = DIR * 2.0 * kPi * turns;
  static constexpr float re = (float)cos_series(ang);
  static constexpr float im = (float)sin_series(ang);
};

template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

// ---- complex arithmetic (paired fp32 pipe where it helps) -----------------
__device__ __forceinline__ float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(-a.y, a.y), make_float2(b.y, b.x)));
}
__device__ __forceinline__ float2 conj(float2 a) { return make_float2(a.x, -a.y); }

// a * W_L^M with a compile-time twiddle
template <int M, int L, int DIR>
__device__ __forceinline__ float2 twc(float2 a) {
  constexpr int m = ((M % L) + L) % L;
  if constexpr (m == 0) {
    return a;
  } else if constexpr (2 * m == L) {
    return make_float2(-a.x, -a.y);
  } else if constexpr (4 * m == L || 4 * m == 3 * L) {
    // W = +-i: DIR * i for m = L/4, -DIR * i for 3L/4
    constexpr int s = (4 * m == L) ? DIR : -DIR;
    return s > 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
  } else if constexpr ((8 * m) % L == 0) {
    // (+-1 +- i)/sqrt(2)
    constexpr float h = 0.70710678118654752440f;
    constexpr float sr = Tw<M, L, DIR>::re > 0 ? 1.f : -1.f;
    constexpr float si = Tw<M, L, DIR>::im > 0 ? 1.f : -1.f;
    return make_float2(h * (sr * a.x - si * a.y), h * (si * a.x + sr * a.y));
  } else {
    constexpr float wr = Tw<M, L, DIR>::re, wi = Tw<M, L, DIR>::im;
    return make_float2(fmaf(a.x, wr, -a.y * wi), fmaf(a.x, wi, a.y * wr));
  }
}

// ---- in-register DFT ---------------------------------------------------------
// Decimation-in-frequency, radix-4 stages (radix 2 last when log2 R is odd).
// On return v[pos] holds frequency freq_at<R>(pos) (a digit reversal that the
// callers fold into their compile-time store indices).
template <int R, int L, int DIR>
__device__ __forceinline__ void dif(float2 (&v)[R]) {
  if constexpr (L > 1) {
    constexpr int r = (L % 4 == 0) ? 4 : 2;
    constexpr int Q = L / r;
    static_for<0, R / L>([&](auto B) {
      constexpr int b = decltype(B)::value * L;
      static_for<0, Q>([&](auto J) {
        constexpr int j = decltype(J)::value;
        if constexpr (r == 4) {
          const float2 a0 = v[b + j], a1 = v[b + j + Q], a2 = v[b + j + 2 * Q], a3 = v[b + j + 3 * Q];
          const float2 y0 = add(a0, a2), y1 = sub(a0, a2), y2 = add(a1, a3);
          const float2 y3 = twc<1, 4, DIR>(sub(a1, a3));
          v[b + j] = add(y0, y2);
          v[b + j + Q] = twc<j, L, DIR>(add(y1, y3));
          v[b + j + 2 * Q] = twc<2 * j, L, DIR>(sub(y0, y2));
          v[b + j + 3 * Q] = twc<3 * j, L, DIR>(sub(y1, y3));
        } else {
          const float2 a0 = v[b + j], a1 = v[b + j + Q];
          v[b + j] = add(a0, a1);
          v[b + j + Q] = twc<j, L, DIR>(sub(a0, a1));
        }
      });
    });
    dif<R, Q, DIR>(v);
  }
}

// frequency held at register position pos after dif<R, R, DIR>
constexpr int freq_at(int R, int pos) {
  int f = 0, mul = 1, L = R;
  while (L > 1) {
    const int r = (L % 4 == 0) ? 4 : 2;
    const int Q = L / r;
    f += (pos / Q) * mul;
    pos %= Q;
    mul *= r;
    L = Q;
  }
  return f;
}

template <int R, int DIR>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
  dif<R, R, DIR>(v);
}

// ---- the batched two-pass transform -----------------------------------------
template <int N>
struct Split {
  static constexpr int R1 = N <= 32 ? N : (1 << ((ilog2(N) + 1) / 2));
  static constexpr int R2 = N / R1;
};

// Named barrier over the NT threads running the transform (BARID 0 =
// __syncthreads; warp-specialised kernels keep their producer warp out).
// BARID < 0: the barrier id is the runtime value rbar (groups of threads that
// run the same code on different barriers share one copy of it).
template <int BARID, int NT>
__device__ __forceinline__ void sync(int rbar = 0) {
  if constexpr (BARID == 0) {
    __syncthreads();
  } else if constexpr (BARID < 0) {
    asm volatile("bar.sync %0, %1;" ::"r"(rbar), "n"(NT) : "memory");
  } else {
    asm volatile("bar.sync %0, %1;" ::"n"(BARID), "n"(NT) : "memory");
  }
}

// Transform C columns.  load(c, n) supplies x[n] of column c; after every
// thread's loads a barrier is passed and loaded() is called by every thread
// (the caller may release its input buffer there); store(c, n, X) receives
// X[n].  tw: table exp(-2 pi i m / N), m < N (shared memory preferred).
// work: N * LDW float2 of shared memory (unused for N <= 32); it may alias the
// memory `load` reads.  Pass 1 maps consecutive threads to consecutive
// columns; pass 2 too (I_FAST2 = false) or to consecutive butterflies of one
// column (I_FAST2 = true: stores of one column contiguous along n; use an odd
// LDW so the column reads are conflict-free).  Called by NT threads (tid in
// [0, NT)).  There is a barrier after the loads and one between the passes;
// the caller synchronises after the call if other threads next read what
// store() wrote, or before the next call's pass-1 loads if they alias work.
// R1SEL overrides the pass-1 radix (0 = Split<N>; e.g. 16 for N = 512 keeps
// pass 1 at 16 registers pairs when the caller is register-limited).
//
// fft_ctx: the same transform, but the output column is resolved once per
// butterfly: ctx = prep(c), then store(ctx, n, X) for each of its outputs
// (e.g. prep returns the column's global pointer, so the unrolled stores are
// single instructions with immediate offsets).
//
// SPLIT2 halves every pass-2 butterfly between two threads (2 C R1 half
// butterflies instead of C R1 full ones, for callers whose NT would otherwise
// leave half the threads idle in pass 2).  With p = 2q + h and the virtual
// index i' = i + h R1 in [0, 2 R1), the DIF radix-2 split of DFT_R2 gives
//   g_r = W_N^{r i'} (y[i + r R1] + W_{2 R1}^{i'} y[i + (r + R2/2) R1]),
//   X[i' + 2 q R1] = DFT_{R2/2}(g)_q,          r, q < R2/2,
// so both halves run the same code (W_{2R1}^{R1} = -1 supplies the sign).
// TW2: `tw` is the pass-2 table laid out by rows, tw[r * tw2_ld + i] =
// W_N^{r i} (r < R2, i < tw2_ld = 2 R1 with SPLIT2, else R1; build_tw2), so
// that the threads of a warp, which take consecutive butterflies i when
// I_FAST2, read consecutive words instead of a stride-r pattern (a 32-way
// bank conflict at r = 16 with the plain table).
template <int N, int R1SEL, bool SPLIT2>
constexpr int tw2_ld() {
  return (R1SEL ? R1SEL : Split<N>::R1) * (SPLIT2 ? 2 : 1);
}
template <int N, int R1SEL, bool SPLIT2>
constexpr int tw2_size() {
  return N <= 32 ? 1 : (N / (R1SEL ? R1SEL : Split<N>::R1)) * tw2_ld<N, R1SEL, SPLIT2>();
}
// tw2[r * L + i] = tw[(r * i) mod N] (tw: exp(-2 pi i m / N), any memory), by
// threads [tid, ..., nthreads)
template <int N, int R1SEL, bool SPLIT2>
__device__ __forceinline__ void build_tw2(float2 *tw2, const float2 *tw, int tid, int nthreads) {
  constexpr int L = tw2_ld<N, R1SEL, SPLIT2>();
  if constexpr (N > 32) {
    for (int e = tid; e < tw2_size<N, R1SEL, SPLIT2>(); e += nthreads) {
      const int r = e / L, i = e - r * L;
      tw2[e] = tw[(r * i) & (N - 1)];
    }
  }
}

// SYNC_STORE: a barrier over the NT threads between the last read of `work`
// and the first store() (one pass-2 butterfly per thread), so that store()
// may write into `work` itself (e.g. a tile for a TMA store).
template <int N, int C, int LDW, int NT, int DIR, int BARID, bool I_FAST2, int R1SEL = 0, bool SPLIT2 = false,
          bool TW2 = false, bool SYNC_STORE = false, typename Load, typename Loaded, typename Prep, typename Store>
__device__ __forceinline__ void fft_ctx(float2 *__restrict__ work, const float2 *__restrict__ tw, int tid,
                                        Load &&load, Loaded &&loaded, Prep &&prep, Store &&store, int rbar = 0) {
  static_assert((N & (N - 1)) == 0 && N >= 2 && N <= 1024, "power-of-two length in [2, 1024]");
  constexpr int R1 = R1SEL ? R1SEL : Split<N>::R1, R2 = N / R1;
  static_assert(R1 <= 32 && R2 <= 32, "two passes of radix <= 32");
  constexpr int TL = TW2 ? tw2_ld<N, R1SEL, SPLIT2>() : 0;   // pass-2 table row length (0: plain table)
  if constexpr (R2 == 1) {
    // single pass: one thread per column
    constexpr int IT = (C + NT - 1) / NT;
    float2 v[IT][R1];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int c = tid + it * NT;
      if (C % NT == 0 || c < C) {
#pragma unroll
        for (int r = 0; r < R1; ++r) v[it][r] = load(c, r);
      }
    }
    sync<BARID, NT>(rbar);
    loaded();
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int c = tid + it * NT;
      if (C % NT == 0 || c < C) {
        dft<R1, DIR>(v[it]);
        const auto ctx = prep(c);
        static_for<0, R1>([&](auto P) {
          constexpr int p = decltype(P)::value;
          store(ctx, freq_at(R1, p), v[it][p]);
        });
      }
    }
  } else {
    // pass 1: all loads of this thread first (the work tile may alias the input)
    constexpr int NB1 = C * R2;
    constexpr int IT1 = (NB1 + NT - 1) / NT;
    float2 v[IT1][R1];
#pragma unroll
    for (int it = 0; it < IT1; ++it) {
      const int b = tid + it * NT;
      if (NB1 % NT == 0 || b < NB1) {
        const int c = b % C, i = b / C;
#pragma unroll
        for (int r = 0; r < R1; ++r) v[it][r] = load(c, i + r * R2);
      }
    }
    sync<BARID, NT>(rbar);
    loaded();
#pragma unroll
    for (int it = 0; it < IT1; ++it) {
      const int b = tid + it * NT;
      if (NB1 % NT == 0 || b < NB1) {
        const int c = b % C, i = b / C;
        dft<R1, DIR>(v[it]);
        static_for<0, R1>([&](auto P) {
          constexpr int p = decltype(P)::value;
          work[(i * R1 + freq_at(R1, p)) * LDW + c] = v[it][p];
        });
      }
    }
    sync<BARID, NT>(rbar);
    if constexpr (SPLIT2) {
      static_assert(R2 >= 4, "split pass 2 needs R2 >= 4");
      constexpr int H = R2 / 2;
      constexpr int NB2 = C * 2 * R1;
      constexpr int IT2 = (NB2 + NT - 1) / NT;
#pragma unroll
      for (int it = 0; it < IT2; ++it) {
        const int b = tid + it * NT;
        if (NB2 % NT == 0 || b < NB2) {
          const int c = I_FAST2 ? b / (2 * R1) : b % C;
          const int ip = I_FAST2 ? b % (2 * R1) : b / C;
          const int i = ip & (R1 - 1);
          float2 e = TW2 ? tw[H * TL + ip] : tw[H * ip];
          if (DIR > 0) e.y = -e.y;
          float2 g[H];
#pragma unroll
          for (int r = 0; r < H; ++r) {
            const float2 t = add(work[(i + r * R1) * LDW + c], mul(work[(i + (r + H) * R1) * LDW + c], e));
            if (r == 0) {
              g[0] = t;
            } else {
              float2 w = TW2 ? tw[r * TL + ip] : tw[r * ip];
              if (DIR > 0) w.y = -w.y;
              g[r] = mul(t, w);
            }
          }
          dft<H, DIR>(g);
          if constexpr (SYNC_STORE) {
            static_assert(NB2 == NT, "SYNC_STORE: one pass-2 butterfly per thread");
            sync<BARID, NT>(rbar);
          }
          const auto ctx = prep(c);
          static_for<0, H>([&](auto P) {
            constexpr int p = decltype(P)::value;
            store(ctx, ip + 2 * freq_at(H, p) * R1, g[p]);
          });
        }
      }
      return;
    }
    // pass 2: butterflies one at a time (reads and writes disjoint per thread)
    constexpr int NB2 = C * R1;
    constexpr int IT2 = (NB2 + NT - 1) / NT;
#pragma unroll
    for (int it = 0; it < IT2; ++it) {
      const int b = tid + it * NT;
      if (NB2 % NT == 0 || b < NB2) {
        const int c = I_FAST2 ? b / R1 : b % C;
        const int i = I_FAST2 ? b % R1 : b / C;
        float2 u[R2];
        u[0] = work[i * LDW + c];
#pragma unroll
        for (int r = 1; r < R2; ++r) {
          float2 w = TW2 ? tw[r * TL + i] : tw[r * i];
          if (DIR > 0) w.y = -w.y;
          u[r] = mul(work[(i + r * R1) * LDW + c], w);
        }
        dft<R2, DIR>(u);
        if constexpr (SYNC_STORE) {
          static_assert(SPLIT2 || NB2 == NT, "SYNC_STORE: one pass-2 butterfly per thread");
          sync<BARID, NT>(rbar);
        }
        const auto ctx = prep(c);
        static_for<0, R2>([&](auto P) {
          constexpr int p = decltype(P)::value;
          store(ctx, i + freq_at(R2, p) * R1, u[p]);
        });
      }
    }
  }
}

template <int N, int C, int LDW, int NT, int DIR, int BARID, bool I_FAST2, int R1SEL = 0, typename Load,
          typename Loaded, typename Store>
__device__ __forceinline__ void fft(float2 *__restrict__ work, const float2 *__restrict__ tw, int tid, Load &&load,
                                    Loaded &&loaded, Store &&store, int rbar = 0) {
  fft_ctx<N, C, LDW, NT, DIR, BARID, I_FAST2, R1SEL>(
      work, tw, tid, load, loaded, [](int c) { return c; }, store, rbar);
}

// consumer threads that give every pass-1 butterfly of a C-column batch its own thread
template <int N, int C>
constexpr int nt_fft() {
  constexpr int nb = C * Split<N>::R2;
  return nb < 32 ? 32 : (nb > 512 ? 512 : nb);
}

}  // namespace sarfft2
