// passb.cu -- opt-in fused pass B (K2 + K3 + K4a, SAR_FUSE=1): see the
// negative result in DESIGN.md section 10.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace sark {
namespace {

// ------------------------------------------------------- fused pass B ----
// K2 + K3 + K4a in one persistent kernel whose intermediates stay in L2.
// Work is grouped by k_x mirror pair p = min(a, nx - a) (the columns of one
// Stolt mirror class live in k_x = p and nx - p), group index G = f*P + p:
//   Y(G): forward y-FFT of the [ny][16 k] tiles of k_x in {p, nx-p} (in place, W0)
//   S(G): filter + Stolt + inverse z-FFT of the classes (p, b), W0 -> W1
//   I(G): inverse y-FFT of the [ny][16 z] tiles of W1 for k_x in {p, nx-p}
// The host-built item list issues Y(s), S(s - LAG), I(s - 2 LAG) at step s,
// so a group's W0/W1 slabs (2 x ny x n_k x 8 B each) are re-read while still
// in L2.  S(G) waits for the Y(G) counter, I(G) for the S(G) counter (the
// producer spins with acquire loads before it issues the TMA reads; writers
// publish with bar + fence + atomicAdd).  Items are taken in list order by
// every persistent CTA, so the smallest unfinished item never waits on a
// later one (deadlock-free with all CTAs resident).  S items discard the
// consumed W0 lines from L2 (discard.global.L2), so W0 is never written back:
// HBM sees one read of W0 and one write of W1.
// Y / I item: y-FFT of one [ny][8] tile (TMA stage) stored in place at base
// (Y: forward, kept in L2 for the S items; I: inverse, streaming stores).
// Ends with a consumer barrier (work is reused by the next item).
template <int NY, int DIR>
__device__ __noinline__ void pb_tile(const float2 *stage, float2 *work, const float2 *twy, float2 *base, size_t row,
                                     int cmax, int tid, uint64_t *empty_st) {
  sarfft2::fft<NY, PB_KC, PB_KC, PB_NT, DIR, 1, false>(
      work, twy, tid, [&](int c, int m) { return stage[m * PB_KC + c]; },
      [&] {
        if (tid == 0) sartma::mbar_arrive(empty_st);
      },
      [&](int c, int m, float2 x) {
        if (c < cmax) {
          if (DIR < 0) base[(size_t)m * row + c] = x;
          else __stcs(base + (size_t)m * row + c, x);
        }
      });
  sarfft2::sync<1, PB_NT>();
}

// S item: Stolt over the in-band bins of each class (filter folded into the
// weights) + inverse z-FFT, W0 columns -> W1 columns.  Ends with a consumer
// barrier.
template <int NY, int NZ, bool DO_IFFT>
__device__ __noinline__ void pb_stolt(const SarDeviceView *vp, unsigned char *sb, size_t hdr_bytes, float2 *work,
                                      const float2 *twz, int tid, int f, int *colofs, int *slo, int *shi,
                                      uint64_t *empty_st, int discard) {
  constexpr int CL = PB_CL, CC = 4 * CL, LD = CC + 1;
  const SarDeviceView &v = *vp;
  const int nk = v.nk, nx = v.nx;
  const K3Hdr<CL> &h = *reinterpret_cast<const K3Hdr<CL> *>(sb);
  const float2 *fin = reinterpret_cast<const float2 *>(sb + hdr_bytes);
  const int nu = h.nused;
  const double rr = v.rref[f] * (1.0 / TWO_PI);
  float2 *fout = work;
  int tot = 0;
#pragma unroll
  for (int cl = 0; cl < CL; ++cl) tot += h.jhi[cl] - h.jlo[cl] + 1;
  for (int idx = tid; idx < tot; idx += PB_NT) {
    int cl = 0, j = idx;
#pragma unroll
    for (int q = 0; q < CL - 1; ++q) {
      const int len = h.jhi[cl] - h.jlo[cl] + 1;
      if (j >= len) {
        j -= len;
        ++cl;
      }
    }
    j += h.jlo[cl];
    const double kr2 = h.kr2[cl];
    int i0 = 0;
    double tau = 0.0;
    const bool ok = stolt_pull(__ldg(v.kz + j), kr2, v.k0, v.inv_dk, v.dk, nk, v.stolt_delta, &i0, &tau);
    float2 wl = make_float2(0.f, 0.f), wu = wl;
    if (ok) {
      const float tt = (float)tau;
      const float2 hl = filter_h(v, __ldg(v.k + i0), kr2, rr, i0);
      const float2 hu = filter_h(v, __ldg(v.k + i0 + 1), kr2, rr, i0 + 1);
      wl = make_float2((1.f - tt) * hl.x, (1.f - tt) * hl.y);
      wu = make_float2(tt * hu.x, tt * hu.y);
    }
    const int nm = h.nmem[cl];
    for (int m = 0; m < nm; ++m) {
      const int sl = h.mslot[cl][m];
      float2 o = make_float2(0.f, 0.f);
      if (ok) o = cmac2(cmul2(wl, fin[sl * nk + i0]), wu, fin[sl * nk + i0 + 1]);
      fout[j * LD + sl] = o;
    }
  }
  if (tid < CC) {
    const bool used = tid < nu;
    colofs[tid] = used ? h.colof[tid] : -1;
    slo[tid] = used ? h.jlo[h.clof[tid]] : NZ;
    shi[tid] = used ? h.jhi[h.clof[tid]] : -1;
  }
  sarfft2::sync<1, PB_NT>();
  if (discard) {
    // the W0 columns of this item are dead: drop them from L2 unwritten
    const int lpc = nk * 8 / 128;
    const float2 *wf = v.w0 + (size_t)f * nx * v.ny * (size_t)nk;
    for (int e = tid; e < nu * lpc; e += PB_NT) {
      const int sl = e / lpc, l = e - sl * lpc;
      discard_l2(reinterpret_cast<const char *>(wf + (size_t)colofs[sl] * nk) + (size_t)l * 128);
    }
  }
  if (tid == 0) sartma::mbar_arrive(empty_st);
  float2 *dst = v.w1 + (size_t)f * nx * v.ny * (size_t)NZ;
  auto load = [&](int c, int m) { return (m >= slo[c] && m <= shi[c]) ? fout[m * LD + c] : make_float2(0.f, 0.f); };
  if constexpr (DO_IFFT) {
    sarfft2::fft<NZ, CC, LD, PB_NT, +1, 1, true>(fout, twz, tid, load, [] {}, [&](int c, int m, float2 x) {
      const int col = colofs[c];
      if (col >= 0) dst[(size_t)col * NZ + m] = x;
    });
  } else {
    for (int i = tid; i < CC * NZ; i += PB_NT) {
      const int sl = i / NZ, z = i - sl * NZ;
      if (sl < nu) dst[(size_t)colofs[sl] * NZ + z] = load(sl, z);
    }
  }
  sarfft2::sync<1, PB_NT>();
}

// item = {type (0 Y, 1 S, 2 I), frame, k_x (Y, I) or p (S), k-chunk / first b / z-chunk}
template <int NY, int NZ, bool DO_IFFT>
__global__ void __launch_bounds__(PB_NT + 32, 2)
    k_passb(const __grid_constant__ SarDeviceView v, const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
            const int4 *__restrict__ items, int nitems, int *__restrict__ cnt, int stop, int discard, int plain) {
  constexpr int CL = PB_CL, CC = 4 * CL, LD = CC + 1;
  constexpr int ROWS = NY < 256 ? NY : 256;
  constexpr int NBOX = NY / ROWS;
  constexpr uint32_t TILE_BYTES = NY * PB_KC * sizeof(float2);
  extern __shared__ __align__(128) unsigned char smq[];
  const int nk = v.nk, nx = v.nx;
  const int P = nx / 2 + 1;
  const size_t hdr_bytes = (sizeof(K3Hdr<CL>) + 15) & ~(size_t)15;
  const size_t stage_bytes = passb_stage_bytes<NY, NZ>(nk);
  unsigned char *ring = smq;
  float2 *work = reinterpret_cast<float2 *>(smq + PB_S * stage_bytes);
  float2 *twy = work + passb_work<NY, NZ>();
  float2 *twz = twy + NY;
  const double *ks = v.k;    // k and k_z tables through L1 (S items only)
  const double *kzs = v.kz;
  __shared__ __align__(8) uint64_t full[PB_S], empty[PB_S];
  __shared__ int colofs[CC], slo[CC], shi[CC];
  const int tid = threadIdx.x;
  for (int i = tid; i < NY; i += PB_NT + 32) twy[i] = v.tw_y[i];
  for (int i = tid; i < NZ; i += PB_NT + 32) twz[i] = v.tw_z[i];
  if (tid == 0) {
    for (int i = 0; i < PB_S; ++i) {
      sartma::mbar_init(&full[i], 1);
      sartma::mbar_init(&empty[i], 1);
    }
    sartma::fence_barrier_init();
  }
  __syncthreads();
  const int nchunk_k = (nk + PB_KC - 1) / PB_KC;
  const int nS = ((v.ny / 2 + 1) + CL - 1) / CL;
  const int FP = v.F * P;
  auto skip = [&](int type) { return (stop == 2 && type != 0) || (stop == 3 && type == 2); };

  if (tid >= PB_NT) {
    // ------------------------------ producer ------------------------------
    if (tid == PB_NT) {
      const int hx = nx / 2 + 1;
      unsigned n = 0;
      for (int t = blockIdx.x; t < nitems; t += gridDim.x) {
        const int4 it = items[t];
        if (skip(it.x)) continue;
        const int st = n % PB_S;
        if (n >= PB_S) sartma::mbar_wait(&empty[st], ((n / PB_S) - 1) & 1);
        unsigned char *sb = ring + st * stage_bytes;
        const int f = it.y;
        if (it.x == 0) {
          sartma::mbar_arrive_expect_tx(&full[st], TILE_BYTES);
#pragma unroll
          for (int bx = 0; bx < NBOX; ++bx)
            sartma::tma_load_3d(sb + bx * ROWS * PB_KC * sizeof(float2), &tm0, it.w * PB_KC, it.z,
                                f * NY + bx * ROWS, &full[st]);
        } else if (it.x == 2 && plain) {
          sartma::mbar_arrive(&full[st]);  // consumers wait for S(G) and load the tile themselves
        } else if (it.x == 2) {
          const int pp = it.z < nx - it.z ? it.z : nx - it.z;
          const int *c = cnt + FP + f * P + pp;
          while (ld_acquire(c) < nS) __nanosleep(64);
          fence_proxy_async_global();
          sartma::mbar_arrive_expect_tx(&full[st], TILE_BYTES);
#pragma unroll
          for (int bx = 0; bx < NBOX; ++bx)
            sartma::tma_load_3d(sb + bx * ROWS * PB_KC * sizeof(float2), &tm1, it.w * PB_KC, it.z,
                                f * NY + bx * ROWS, &full[st]);
        } else {
          const int pp = it.z;
          const int nkx = (pp == 0 || 2 * pp == nx) ? 1 : 2;
          const int *c = cnt + f * P + pp;
          if (!plain) {
            while (ld_acquire(c) < nkx * nchunk_k) __nanosleep(64);
            fence_proxy_async_global();
          }
          K3Hdr<CL> &h = *reinterpret_cast<K3Hdr<CL> *>(sb);
          float2 *fin = reinterpret_cast<float2 *>(sb + hdr_bytes);
          int nc = 0;
          for (int cl = 0; cl < CL; ++cl) {
            const int b = it.w + cl;
            h.nmem[cl] = 0;
            h.kr2[cl] = 0.0;
            h.jlo[cl] = 0;
            h.jhi[cl] = -1;
            if (b >= v.ny / 2 + 1) continue;
            const SarClass &c = v.cls[b * hx + pp];
            h.kr2[cl] = c.kr2;
            h.jlo[cl] = c.jlo;
            h.jhi[cl] = c.jhi;
            for (int m = 0; m < c.nmem; ++m) {
              h.mslot[cl][h.nmem[cl]++] = nc;
              h.clof[nc] = cl;
              h.colof[nc++] = c.col[m];
            }
          }
          h.nused = nc;
          h.f = f;
          const float2 *wf = v.w0 + (size_t)f * nx * v.ny * (size_t)nk;
          if (plain) {
            sartma::mbar_arrive(&full[st]);  // consumers wait for Y(G) and load the columns
          } else {
            sartma::mbar_arrive_expect_tx(&full[st], (uint32_t)nc * (uint32_t)nk * 8u);
            for (int sl = 0; sl < nc; ++sl)
              sartma::bulk_g2s(fin + sl * nk, wf + (size_t)h.colof[sl] * nk, (uint32_t)nk * 8u, &full[st]);
          }
        }
        ++n;
      }
    }
    return;
  }
  // ------------------------------ consumers ------------------------------
  unsigned n = 0;
  for (int t = blockIdx.x; t < nitems; t += gridDim.x) {
    const int4 it = items[t];
    if (skip(it.x)) continue;
    const int st = n % PB_S;
    sartma::mbar_wait(&full[st], (n / PB_S) & 1);
    unsigned char *sb = ring + st * stage_bytes;
    const int f = it.y;
    if (plain && it.x != 0) {
      // wait for the producing items, then load through L2 with ordinary
      // (coherent) loads: no TMA read of lines this kernel just wrote
      if (tid == 0) {
        const int pp = it.x == 2 ? (it.z < nx - it.z ? it.z : nx - it.z) : it.z;
        const int nkx = (pp == 0 || 2 * pp == nx) ? 1 : 2;
        const int *c = it.x == 2 ? cnt + FP + f * P + pp : cnt + f * P + pp;
        const int target = it.x == 2 ? nS : nkx * nchunk_k;
        while (ld_acquire(c) < target) __nanosleep(64);
      }
      sarfft2::sync<1, PB_NT>();
      if (it.x == 2) {
        const float4 *src = reinterpret_cast<const float4 *>(v.w1 + ((size_t)f * NY * nx + it.z) * (size_t)v.nz +
                                                             it.w * PB_KC);
        float4 *dstt = reinterpret_cast<float4 *>(sb);
        const size_t row4 = (size_t)nx * v.nz / 2;
        for (int e = tid; e < NY * PB_KC / 2; e += PB_NT) {
          const int r = e / (PB_KC / 2), q = e - r * (PB_KC / 2);
          dstt[e] = __ldcg(src + r * row4 + q);
        }
      } else {
        const K3Hdr<CL> &h = *reinterpret_cast<const K3Hdr<CL> *>(sb);
        float4 *fin4 = reinterpret_cast<float4 *>(sb + hdr_bytes);
        const float2 *wf = v.w0 + (size_t)f * nx * v.ny * (size_t)nk;
        const int h2 = nk / 2;
        for (int e = tid; e < h.nused * h2; e += PB_NT) {
          const int sl = e / h2, i = e - sl * h2;
          fin4[e] = __ldcg(reinterpret_cast<const float4 *>(wf + (size_t)h.colof[sl] * nk) + i);
        }
      }
      sarfft2::sync<1, PB_NT>();
    }
    if (it.x != 1) {
      const int inner = it.x == 0 ? nk : v.nz;
      float2 *base = (it.x == 0 ? v.w0 : v.w1) + ((size_t)f * NY * nx + it.z) * (size_t)inner + it.w * PB_KC;
      if (it.x == 0) {
        pb_tile<NY, -1>(reinterpret_cast<const float2 *>(sb), work, twy, base, (size_t)nx * inner,
                        inner - it.w * PB_KC, tid, &empty[st]);
        if (tid == 0) {
          __threadfence();
          fence_proxy_async_global();
          const int pp = it.z < nx - it.z ? it.z : nx - it.z;
          atomicAdd(cnt + f * P + pp, 1);
        }
      } else {
        pb_tile<NY, +1>(reinterpret_cast<const float2 *>(sb), work, twy, base, (size_t)nx * inner,
                        inner - it.w * PB_KC, tid, &empty[st]);
      }
    } else {
      pb_stolt<NY, NZ, DO_IFFT>(&v, sb, hdr_bytes, work, twz, tid, f, colofs, slo, shi, &empty[st], discard);
      if (tid == 0) {
        __threadfence();
        fence_proxy_async_global();
        atomicAdd(cnt + FP + f * P + it.z, 1);
      }
    }
    ++n;
  }
}


}  // namespace

#define SAR_PASSB_PAIRS(X) X(64, 16) X(128, 64) X(128, 128) X(256, 128) X(256, 256) X(512, 512)

bool passb_supported(const SarDeviceView &v) {
  if ((v.nk & 1) || v.nk > 512 || v.ny > 512) return false;
#define X(A, B) \
  if (v.ny == A && v.nz == B) return passb_smem<A, B>(v.nk) <= 227 * 1024;
  SAR_PASSB_PAIRS(X)
#undef X
  return false;
}

cudaError_t launch_passb(const SarDeviceView &v, const CUtensorMap *tm0, const CUtensorMap *tm1, const int4 *items,
                         int nitems, int *cnt, int stop, bool discard, cudaStream_t s, int num_sms) {
  const int plain = getenv("SAR_PB_PLAIN") ? 1 : 0;
  cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)2 * v.F * (v.nx / 2 + 1) * sizeof(int), s);
  if (e != cudaSuccess) return e;
#define X(A, B)                                                                                         \
  if (v.ny == A && v.nz == B) {                                                                         \
    const size_t smem = passb_smem<A, B>(v.nk);                                                         \
    auto kern = stop == 3 ? k_passb<A, B, false> : k_passb<A, B, true>;                                 \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);             \
    if (e != cudaSuccess) return e;                                                                     \
    int occ = 0; /* every CTA must be resident: the items wait on each other */                        \
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PB_NT + 32, smem);                   \
    if (e != cudaSuccess) return e;                                                                     \
    if (occ < 1) return cudaErrorInvalidConfiguration;                                                  \
    const int maxg = num_sms * occ;                                                                     \
    const int grid = nitems < maxg ? nitems : maxg;                                                     \
    kern<<<grid, PB_NT + 32, smem, s>>>(v, *tm0, *tm1, items, nitems, cnt, stop, discard ? 1 : 0, plain); \
    return cudaGetLastError();                                                                          \
  }
  SAR_PASSB_PAIRS(X)
#undef X
  return cudaErrorInvalidValue;
}


// Fused pass B: decide, build the item list (see k_passb) and allocate it with
// the dependency counters.  Returns SAR_OK with p->fused = false when the
// geometry is not covered.
}  // namespace sark

int sar_setup_passb(sar_plan *p) {
  using namespace sark;
  const SarDeviceView &v = p->v;
  p->fused = false;
  // opt-in (SAR_FUSE=1): measured slower than the unfused kernels on B200 --
  // the dirty W0/W1 slabs do not survive in L2 between producer and consumer
  // items (DRAM writes 3.3 GB instead of 1.07 GB at Large), see DESIGN.md
  if (v.F == 0 || v.mode2d || v.nufft || !getenv("SAR_FUSE") || !p->tma_pb || !passb_supported(v)) return SAR_OK;
  const int P = v.nx / 2 + 1;
  const int nchunk_k = (v.nk + PB_KC - 1) / PB_KC, nchunk_z = (v.nz + PB_KC - 1) / PB_KC;
  const int GT = v.F * P;
  auto kxs = [&](int pp, int *o) {
    o[0] = pp;
    o[1] = v.nx - pp;
    return (pp == 0 || 2 * pp == v.nx) ? 1 : 2;
  };
  // lag (in steps) between Y(G) and S(G) and between S(G) and I(G): at least
  // three waves of CTAs worth of items, at most ~48 MB of live slabs in L2
  const int per_step = 2 * nchunk_k + (v.ny / 2 + 1 + PB_CL - 1) / PB_CL + 2 * nchunk_z;
  const double slab = 2.0 * v.ny * ((double)v.nk + v.nz) * sizeof(float2);
  int lag = (3 * 2 * p->num_sms + per_step - 1) / per_step;
  const int lag_max = (int)(48e6 / slab);
  if (lag > lag_max) lag = lag_max;
  if (lag < 1) lag = 1;
  std::vector<int4> items;
  for (int st = 0; st < GT + 2 * lag; ++st) {
    int kx[2];
    if (st < GT) {
      const int f = st / P, pp = st % P;
      const int nkx = kxs(pp, kx);
      for (int q = 0; q < nkx; ++q)
        for (int c = 0; c < nchunk_k; ++c) items.push_back(make_int4(0, f, kx[q], c));
    }
    if (st - lag >= 0 && st - lag < GT) {
      const int g = st - lag, f = g / P, pp = g % P;
      for (int b0 = 0; b0 < v.ny / 2 + 1; b0 += PB_CL) items.push_back(make_int4(1, f, pp, b0));
    }
    if (st - 2 * lag >= 0 && st - 2 * lag < GT) {
      const int g = st - 2 * lag, f = g / P, pp = g % P;
      const int nkx = kxs(pp, kx);
      for (int q = 0; q < nkx; ++q)
        for (int c = 0; c < nchunk_z; ++c) items.push_back(make_int4(2, f, kx[q], c));
    }
  }
  p->n_items = (int)items.size();
  if (cudaMalloc(&p->d_items, items.size() * sizeof(int4)) != cudaSuccess ||
      cudaMalloc(&p->d_cnt, (size_t)2 * GT * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    return SAR_ERR_OOM;
  }
  if (cudaMemcpy(p->d_items, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice) != cudaSuccess)
    return SAR_ERR_CUDA;
  p->passb_discard = ((size_t)v.nk * 8) % 128 == 0 && !getenv("SAR_NO_DISCARD");
  p->fused = true;
  return SAR_OK;
}

namespace sark {

}  // namespace sark
