// k4.cu -- K4b: inverse x-FFT + |.|/(nx ny nz) + integer rolls (IFT_3D of
// Eq. (14); readings R8, R11), W1 -> image.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace sark {
namespace {

// |o| by the SFU square root (sqrt.approx: one MUFU, relative error <= 2^-23,
// exact 0 at 0) instead of the IEEE sqrtf sequence with its slow-path call
__device__ __forceinline__ float fast_abs(float2 o) {
  const float p = fmaf(o.x, o.x, o.y * o.y);
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
  return r;
}


// SAR_REPORT_PEAK: warp max of the magnitudes a thread wrote, one atomic per
// warp (non-negative floats order like their bit patterns)
__device__ __forceinline__ void report_peak(const SarDeviceView &v, int f, float pk) {
  if (!v.peak) return;
  const unsigned b = __reduce_max_sync(0xffffffffu, __float_as_uint(pk));
  if ((threadIdx.x & 31) == 0 && b) atomicMax(v.peak + v.f0 + f, b);
}

// Warp-specialised persistent K4b (nx <= 512, n_z even): [nx][16 z] tiles of
// W1 row y stream through an S-stage TMA ring; the consumers run the inverse
// x-FFT (pass 2 mapped so that one warp owns 32 consecutive x of one z) and
// write |o|/(nx ny nz) (or the scaled complex value) straight into the rolled
// image rows (reading R8, R11): coalesced 128-byte segments, no transpose
// buffer.
// consumer threads and pass split of the x-IFFT: one thread per pass-1
// butterfly (512 threads with the split pass 2, as in K2, measured slower:
// 0.347 vs 0.314 ms on Large)
template <int NX>
struct K4bFft {
  static constexpr bool BIG = false;
  static constexpr int NTC = BIG ? 512 : sarfft2::nt_fft<NX, KC>();
  static constexpr int R1S = BIG ? 16 : 0;
  static constexpr int TWN = sarfft2::tw2_size<NX, R1S, BIG>() > NX ? sarfft2::tw2_size<NX, R1S, BIG>() : NX;
};
template <int NX, bool CPLX>
constexpr size_t k4b2_smem() {
  return ((size_t)2 * NX * KC + (size_t)NX * (KC + 1) + K4bFft<NX>::TWN) * sizeof(float2);
}
template <int NX>
constexpr int k4b2_ctas() {
  return (int)((200 * 1024) / k4b2_smem<NX, false>()) < 1 ? 1 : (int)((200 * 1024) / k4b2_smem<NX, false>());
}

// SLAB: tm is a 4-D map over the received blocks [G][ny][nx'][nz'] of the
// slab exchange #2 (box {16 z, nx', 1, G} = one [nx][16] tile), so stage 3
// needs no unpack pass.
// PEAK: SAR_REPORT_PEAK plans (the running max costs one instruction per voxel)
template <int NX, bool CPLX, bool SLAB, bool PEAK>
__global__ void __launch_bounds__(K4bFft<NX>::NTC + 32)
    k4_xifft_mag2(const SarDeviceView v, const __grid_constant__ CUtensorMap tm, void *__restrict__ img, int nzc,
                  int nitems) {
  using FT = K4bFft<NX>;
  constexpr int NTC = FT::NTC;
  constexpr int S = 2;
  constexpr int ROWS = NX < 256 ? NX : 256;
  constexpr int NBOX = NX / ROWS;
  constexpr uint32_t TILE_BYTES = NX * KC * sizeof(float2);
  using OT = typename std::conditional<CPLX, float2, float>::type;
  extern __shared__ __align__(128) float2 smk[];
  float2 *ring = smk;                          // [S][NX][16]
  float2 *work = smk + (size_t)S * NX * KC;    // [NX][17]
  float2 *tw = work + (size_t)NX * (KC + 1);   // [NX]
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x;
  sarfft2::build_tw2<NX, FT::R1S, FT::BIG>(tw, v.tw_x, tid, NTC + 32);   // pass-2 rows
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
        const int zc = item % nzc, fy = item / nzc;  // fy = f*ny + y
        sartma::mbar_arrive_expect_tx(&full[st], TILE_BYTES);
        if constexpr (SLAB) {
          sartma::tma_load_4d_stream<8>(ring + (size_t)st * NX * KC, &tm, zc * KC, 0, fy, 0, &full[st]);
        } else {
#pragma unroll
          for (int bx = 0; bx < NBOX; ++bx)
            sartma::tma_load_3d_stream<8>(ring + (size_t)st * NX * KC + bx * ROWS * KC, &tm, zc * KC, bx * ROWS, fy, &full[st]);
        }
      }
    }
    return;
  }
  const int nz = v.nz;
  const int rx = ((v.roll_x % NX) + NX) % NX;
  const int ry = ((v.roll_y % v.ny) + v.ny) % v.ny;
  const float sc = v.img_scale;
  const size_t zstride = (size_t)v.ny * NX;
  unsigned n = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
    const int st = n % S;
    sartma::mbar_wait(&full[st], (n / S) & 1);
    const int zc = item % nzc, fy = item / nzc;
    const int f = fy / v.ny, y = fy - f * v.ny;
    int iy = y - ry;
    if (iy < 0) iy += v.ny;
    OT *outp = reinterpret_cast<OT *>(img) + ((size_t)f * v.nz_img * v.ny + iy) * NX;
    const float2 *stage = ring + (size_t)st * NX * KC;
    float pk = 0.f;
    // the image row of z-slot c is resolved once per butterfly (prep), so a
    // store is the x roll plus one STG
    sarfft2::fft_ctx<NX, KC, KC + 1, NTC, +1, 1, true, FT::R1S, FT::BIG, (NX > 32)>(
        work, tw, tid, [&](int c, int m) { return stage[m * KC + c]; },
        [&] {
          if (tid == 0) sartma::mbar_arrive(&empty[st]);
        },
        [&](int c) -> OT * {
          const int z = zc * KC + c;
          if (z >= nz) return nullptr;
          int m = z + v.z_off + v.zroll;
          if (m >= v.nz_img) m -= v.nz_img;
          return outp + (size_t)m * zstride;
        },
        [&](OT *rowp, int a, float2 o) {
          if (rowp) {
            const int ix = (a - rx) & (NX - 1);
            const float mag = fast_abs(o) * sc;
            if constexpr (PEAK) pk = fmaxf(pk, mag);
            SAR_ASSERT(v.img_elems == 0 || (rowp + ix >= reinterpret_cast<OT *>(img) &&
                                             rowp + ix < reinterpret_cast<OT *>(img) + v.img_elems));
            if constexpr (CPLX) {
              __stcs(reinterpret_cast<float2 *>(rowp) + ix, make_float2(o.x * sc, o.y * sc));
            } else {
              __stcs(reinterpret_cast<float *>(rowp) + ix, mag);
            }
          }
        });
    if constexpr (PEAK) report_peak(v, f, pk);
  }
}

// --------------------------------------------------------------- K4b ------
// One CTA = (z chunk, image row y (pre-roll), frame).  Tile [NX][17]: the odd
// stride makes both the FFT passes and the transposed read conflict-free.
template <int NX, bool CPLX>
__global__ void __launch_bounds__(nt_for(NX), minb_for(NX))
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
  float pk = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int zz = item / NX, ix = item - zz * NX;
    const int z = zbase + zz;
    if (z >= nz) continue;
    int m = z + v.z_off + v.zroll;
    if (m >= v.nz_img) m -= v.nz_img;
    const int xs = (ix + rx) & (NX - 1);
    const float2 o = tile[xs * LD + zz];
    const size_t off = ((size_t)(f * v.nz_img + m) * v.ny + iy) * NX + ix;
    SAR_ASSERT(v.img_elems == 0 || off < v.img_elems);
    const float mag = fast_abs(o) * sc;
    pk = fmaxf(pk, mag);
    if constexpr (CPLX) {
      reinterpret_cast<float2 *>(img)[off] = make_float2(o.x * sc, o.y * sc);
    } else {
      reinterpret_cast<float *>(img)[off] = mag;
    }
  }
  report_peak(v, f, pk);
}

template <typename K>
cudaError_t launch_img(K kernel, dim3 grid, int nt, size_t smem, cudaStream_t s, const SarDeviceView &v,
                       void *img) {
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, nt, smem, s>>>(v, img);
  return cudaGetLastError();
}


}  // namespace

cudaError_t launch_k4b(const SarDeviceView &v, void *img, bool cplx, cudaStream_t s, const CUtensorMap *tm,
                       int num_sms, bool slab4d) {
  if (slab4d && !(tm && v.nx <= 512)) return cudaErrorInvalidValue;
  if (tm && v.nx <= 512) {
    const int nzc = (v.nz + KC - 1) / KC;
    const int nitems = nzc * v.ny * v.F;
    switch (v.nx) {
#define X(N)                                                                                           \
  case N: {                                                                                            \
    auto kern = cplx ? k4_xifft_mag2<N, true, false, false> : k4_xifft_mag2<N, false, false, false>;   \
    if (v.peak) kern = cplx ? k4_xifft_mag2<N, true, false, true> : k4_xifft_mag2<N, false, false, true>; \
    if (slab4d) kern = cplx ? k4_xifft_mag2<N, true, true, false> : k4_xifft_mag2<N, false, true, false>; \
    constexpr size_t smem = k4b2_smem<N, false>();                                                     \
    if (smem > 40 * 1024) {                                                                            \
      cudaError_t e0 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (e0 != cudaSuccess) return e0;                                                                \
    }                                                                                                  \
    const int occ = resident_ctas((const void *)kern, K4bFft<N>::NTC + 32, smem);                      \
    const int maxg = num_sms * (occ < k4b2_ctas<N>() ? occ : k4b2_ctas<N>());                                                         \
    cudaError_t e = launch_ex(kern, dim3(nitems < maxg ? nitems : maxg), dim3(K4bFft<N>::NTC + 32), smem, s, \
                               v, *tm, img, nzc, nitems);                                              \
    if (e != cudaSuccess) return e;                                                                    \
    return cudaGetLastError();                                                                         \
  }
      X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512)
#undef X
    }
  }
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



}  // namespace sark
