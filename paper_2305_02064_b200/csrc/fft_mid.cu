// fft_mid.cu -- K2 / K4a: FFT along the middle (y) axis, forward on W0 and
// inverse on W1 (FT_2D / IFT_3D of Eq. (14)).

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace sark {
namespace {

// ------------------------------------------------------------ K2 / K4a ----
// FFT along the middle (y) axis of a [F][N][nx][inner] complex volume for one
// (chunk of 16 along `inner`, column a, frame f).
// live(m, lb): spectral row m (signed index m_s) of a column whose live rows
// are |m_s| <= lb (lb < 0: none); the rows of evanescent / out-of-window
// columns (host class table) are never read
__device__ __forceinline__ bool row_live(int m, int n, int lb) { return m <= lb || n - m <= lb; }

template <int N, int DIR>
__global__ void __launch_bounds__(nt_for(N), minb_for(N))
    k_fft_mid(float2 *__restrict__ data, const float2 *__restrict__ tw, int nx, int inner,
              const int *__restrict__ liveb) {
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
  const int lb = liveb ? liveb[a] : N;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int cc = item & (KC - 1), b = item >> 4;
    const int c = cbase + cc;
    // inverse (K4a): rows of skipped columns are zero; forward (K2): all rows read
    tile[item] = c < inner && (DIR < 0 || row_live(b, N, lb)) ? base[b * row + c] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  sarfft::tile_fft<N, KC, KC, NT, DIR>(tile, tw, tid);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int cc = item & (KC - 1), b = item >> 4;
    const int c = cbase + cc;
    // forward (K2): rows no later stage reads are not stored
    if (c < inner && (DIR > 0 || row_live(b, N, lb))) base[b * row + c] = tile[item];
  }
}

// Warp-specialised persistent mid-axis FFT (K2 / K4a, ny <= 512, `inner`
// even).  A producer warp streams [N][16] tiles (3-D TMA boxes {16 inner, 1
// column, <=256 rows}) into an S-stage mbarrier ring; NTC consumer threads run
// the two-pass register FFT (fft_reg.cuh), hand the stage back right after
// the pass-1 loads, and store the transformed rows straight to global memory
// (each warp store = two full 128-byte lines).
#ifndef MID_S_SMALL
#define MID_S_SMALL 6   // ring stages of the mid-axis FFT below N = 256 (Realtime K2 0.41 -> 0.38 ms, K4a 0.20 -> 0.17)
#endif
template <int N>
constexpr int mid2_stages() { return N >= 256 ? 2 : MID_S_SMALL; }
template <int N>
constexpr size_t mid2_smem() {
  return ((size_t)mid2_stages<N>() * N * KC + (size_t)N * KC + N) * sizeof(float2);
}
template <int N>
constexpr int mid2_ctas() {
  return (int)((200 * 1024) / mid2_smem<N>()) < 1 ? 1 : (int)((200 * 1024) / mid2_smem<N>());
}

// consumer threads: 512 at N = 512 (pass 1 as 16 x 32, pass 2 split between
// thread pairs: 512 butterflies in both passes)
template <int N>
constexpr int mid2_ntc() { return N == 512 ? 512 : sarfft2::nt_fft<N, KC>(); }

// TMA box rows: the forward transform (K2) reads whole columns in <= 256-row
// boxes; the inverse (K4a) reads only the boxes of 32 rows that hold live rows
template <int N, int DIR>
constexpr int mid2_rows() { return DIR < 0 ? (N < 256 ? N : 256) : (N < K4A_ROWS ? N : K4A_ROWS); }

// TST: the transformed tile is written back by TMA bulk-tensor stores of
// [32 rows][16] boxes (tm_st) from the work tile instead of one STG per
// element (the per-element 64-bit address arithmetic was a fifth of the
// kernel's instructions); K2 stores only the boxes that hold live rows.
template <int N, int DIR, bool SLAB, bool TST>
__global__ void __launch_bounds__(mid2_ntc<N>() + 32)
    k_fft_mid2(const __grid_constant__ CUtensorMap tm, float2 *__restrict__ data, const float2 *__restrict__ twg,
               int nx, int inner, int nchunk, int nitems, const MidSlabOut so, const int *__restrict__ liveb,
               int oob_row, const __grid_constant__ CUtensorMap tm_st) {
  constexpr int NTC = mid2_ntc<N>();
  constexpr int S = mid2_stages<N>();
  constexpr int ROWS = mid2_rows<N, DIR>();
  constexpr int NBOX = N / ROWS;
  constexpr uint32_t TILE_BYTES = N * KC * sizeof(float2);
  extern __shared__ __align__(128) float2 smm[];
  float2 *ring = smm;                         // [S][N][16]
  float2 *work = smm + (size_t)S * N * KC;    // [N][16]
  float2 *tw = work + (size_t)N * KC;         // [N]
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x;
  for (int i = tid; i < N; i += NTC + 32) tw[i] = twg[i];
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      sartma::mbar_init(&full[i], 1);
      sartma::mbar_init(&empty[i], 1);
    }
    sartma::fence_barrier_init();
  }
  __syncthreads();
  if (tid >= NTC) {
    if (tid == NTC) {
      unsigned n = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
        const int st = n % S;
        if (n >= S) sartma::mbar_wait(&empty[st], ((n / S) - 1) & 1);
        const int chunk = item % nchunk, rest = item / nchunk;
        const int a = rest % nx, f = rest / nx;
        if (DIR > 0 && liveb) {
          // boxes that hold a live row (|m_s| <= lb) are read; the others are
          // requested out of bounds (row F*N), which TMA fills with zeros
          // without touching memory.  Every row of a box read here was
          // written by K3 (its class list covers whole boxes, plan.cpp).
          const int lb = liveb[a];
          sartma::mbar_arrive_expect_tx(&full[st], TILE_BYTES);
#pragma unroll
          for (int bx = 0; bx < NBOX; ++bx) {
            const bool live = lb >= 0 && (bx * ROWS <= lb || (bx + 1) * ROWS - 1 >= N - lb);
            sartma::tma_load_3d_stream<2>(ring + (size_t)st * N * KC + bx * ROWS * KC, &tm, chunk * KC, a,
                                live ? f * N + bx * ROWS : oob_row, &full[st]);
          }
        } else {
          sartma::mbar_arrive_expect_tx(&full[st], TILE_BYTES);
#pragma unroll
          for (int bx = 0; bx < NBOX; ++bx)
            sartma::tma_load_3d_stream<2>(ring + (size_t)st * N * KC + bx * ROWS * KC, &tm, chunk * KC, a,
                                f * N + bx * ROWS, &full[st]);
        }
      }
    }
    return;
  }
  const size_t row = SLAB ? (size_t)nx * so.nzl : (size_t)nx * inner;
  unsigned n = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
    const int st = n % S;
    sartma::mbar_wait(&full[st], (n / S) & 1);
    const int chunk = item % nchunk, rest = item / nchunk;
    const int a = rest % nx, f = rest / nx;
    const float2 *stage = ring + (size_t)st * N * KC;
    float2 *base;
    if constexpr (SLAB) {
      const int h = chunk * KC / so.nzl;
      base = reinterpret_cast<float2 *>(so.d[h]) + (size_t)a * so.nzl + (chunk * KC - h * so.nzl);
    } else {
      base = data + ((size_t)f * N * nx + a) * (size_t)inner + chunk * KC;
    }
    const int cmax = inner - chunk * KC;
    // forward (K2): the live rows (m + lb) mod N < 2 lb + 1 are stored (one
    // add, and, compare per store; the two-sided test costs spills)
    const int lb = (DIR < 0 && liveb) ? liveb[a] : N;
    const unsigned span = lb < 0 ? 0u : (2 * lb + 1 >= N ? (unsigned)N : (unsigned)(2 * lb + 1));
    const int lbo = lb < 0 ? 0 : lb;
    if constexpr (TST) {
      // the previous tile's bulk stores have finished reading `work` before
      // this tile's pass 1 (after its barrier) writes it
      if (tid == 0) sartma::bulk_wait_read0();
    }
    sarfft2::fft_ctx<N, KC, KC, NTC, DIR, 1, false, (N == 512 ? 16 : 0), (N == 512), false, TST>(
        work, tw, tid, [&](int c, int m) { return stage[m * KC + c]; },
        [&] {
          if (tid == 0) sartma::mbar_arrive(&empty[st]);
        },
        [](int c) { return c; },
        [&](int c, int m, float2 v) {
          if constexpr (TST) {
            work[m * KC + c] = v;
          } else {
            if (c < cmax && (DIR > 0 || (unsigned)((m + lbo) & (N - 1)) < span)) {
              SAR_ASSERT(SLAB || (base + (size_t)m * row + c >= data &&
                                  base + (size_t)m * row + c < data + (size_t)(nitems / nchunk / nx) * N * nx * inner));
              st_mid(base + (size_t)m * row + c, v);
            }
          }
        });
    if constexpr (TST) {
      constexpr int SR = N < 32 ? N : 32;
      sartma::fence_proxy_async();   // the tile's generic writes, then the bulk (async proxy) reads
      sarfft2::sync<1, NTC>();
      if (tid == 0) {
#pragma unroll
        for (int bx = 0; bx < N / SR; ++bx) {
          const bool live = DIR > 0 || (lb >= 0 && (bx * SR <= lb || (bx + 1) * SR - 1 >= N - lb));
          if (live) sartma::tma_store_3d(&tm_st, chunk * KC, a, f * N + bx * SR, work + bx * SR * KC);
        }
        sartma::bulk_commit();
      }
    }
  }
  if constexpr (TST) {
    if (tid == 0) sartma::bulk_wait0();
  }
}


}  // namespace

template <int DIR>
cudaError_t launch_mid(float2 *data, const float2 *tw, int F, int ny, int nx, int inner, cudaStream_t s,
                       const CUtensorMap *tm, int num_sms, const MidSlabOut *so, const int *liveb,
                       const CUtensorMap *tm_st) {
  const MidSlabOut off{};
  if (so && !(tm && ny <= 512 && F == 1 && so->nzl % KC == 0)) return cudaErrorInvalidValue;
  if (tm && ny <= 512) {
    const int nchunk = (inner + KC - 1) / KC;
    const int nitems = nchunk * nx * F;
    switch (ny) {
#define X(N)                                                                                       \
  case N: {                                                                                        \
    void (*kern)(const CUtensorMap, float2 *, const float2 *, int, int, int, int, const MidSlabOut,    \
                 const int *, int, const CUtensorMap) = k_fft_mid2<N, DIR, false, false>;           \
    if (so) kern = k_fft_mid2<N, DIR, true, false>;                                                \
    else if (tm_st && N >= 256) kern = k_fft_mid2<N, DIR, false, (N >= 256)>;                      \
    constexpr size_t smem = mid2_smem<N>();                                                        \
    if (smem > 40 * 1024) {                                                                        \
      cudaError_t e0 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (e0 != cudaSuccess) return e0;                                                            \
    }                                                                                              \
    const int occ = resident_ctas((const void *)kern, mid2_ntc<N>() + 32, smem);                  \
    const int maxg = num_sms * (occ < mid2_ctas<N>() ? occ : mid2_ctas<N>());                                                     \
    cudaError_t e = launch_ex(kern, dim3(nitems < maxg ? nitems : maxg), dim3(mid2_ntc<N>() + 32), smem, s, \
                               *tm, data, tw, nx, inner, nchunk, nitems, so ? *so : off, liveb, 1 << 30, \
                               tm_st ? *tm_st : *tm);                                              \
    if (e != cudaSuccess) return e;                                                                \
    return cudaGetLastError();                                                                     \
  }
      X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512)
#undef X
    }
    return cudaErrorInvalidValue;
  }
  dim3 grid((inner + KC - 1) / KC, nx, F);
  const size_t smem = (size_t)ny * KC * sizeof(float2);
  switch (ny) {
#define X(N)                                                                                       \
  case N: {                                                                                        \
    auto kern = k_fft_mid<N, DIR>;                                                                 \
    if (smem > 40 * 1024) {                                                                        \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (e != cudaSuccess) return e;                                                              \
    }                                                                                              \
    kern<<<grid, nt_for(N), smem, s>>>(data, tw, nx, inner, liveb);                                \
    return cudaGetLastError();                                                                     \
  }
    SAR_SIZES(X)
#undef X
  }
  return cudaErrorInvalidValue;
}


template cudaError_t launch_mid<-1>(float2 *, const float2 *, int, int, int, int, cudaStream_t, const CUtensorMap *, int,
                                    const MidSlabOut *, const int *, const CUtensorMap *);
template cudaError_t launch_mid<+1>(float2 *, const float2 *, int, int, int, int, cudaStream_t, const CUtensorMap *, int,
                                    const MidSlabOut *, const int *, const CUtensorMap *);

}  // namespace sark
