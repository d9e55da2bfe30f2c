// k3.cu -- K3: RMA filter + Stolt resampling + inverse z-FFT (Eqs. (13)-(14),
// P:204-226; readings R2-R5, R9), W0 -> W1; the 2-D plane sum (reading R18);
// the device Stolt index table for the bit-exact tests.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace sark {
namespace {

// K3, one small CTA per CL mirror classes (CL = 1 at n_z = 512: the <= 4
// columns (+-a, +-b) that share k_r^2).  128 threads and ~40 KB of shared
// memory, so ~5 CTAs are resident per SM and the hardware overlaps their
// load / fp64 / FFT phases.  Steps: (1) stream the member columns in (n_k
// contiguous samples each); (2) filter H = k_z e^{+j k_z R_ref}/P on the
// source grid, once per class (readings R2-R4); (3) Stolt pull with the
// filter folded into the two complex interpolation weights, decisions bit-exact
// (R5, R9), once per (class, j), applied to every member; (4) inverse z-FFT
// (two-pass register FFT, the Stolt tile doubles as its work tile) whose
// pass 2 stores each column contiguously [col][z].
constexpr int K3C_NT = 128;
template <int NZ>
constexpr int k3c_r1() { return NZ == 512 ? 16 : sarfft2::Split<NZ>::R1; }
template <int NZ>
constexpr int k3c_cl() {
  constexpr int cc = K3C_NT / (NZ / k3c_r1<NZ>());
  return cc / 4 > 8 ? 8 : (cc / 4 < 1 ? 1 : cc / 4);
}
template <int NZ, int CL>
size_t k3c_smem(int nk) {
  return ((size_t)4 * CL * nk + (size_t)NZ * (4 * CL + 1) +
          sarfft2::tw2_size<NZ, (NZ == 512 ? 16 : 0), false>()) * sizeof(float2);
}

// CL classes per CTA: k3c_cl<NZ>() normally, 1 when n_k is so large that
// CL whole columns do not fit in shared memory (up to SAR_MAX_NK)
template <int NZ, bool DO_IFFT, int CL>
__global__ void __launch_bounds__(K3C_NT, 8) k3_class(const SarDeviceView v) {
  constexpr int CC = 4 * CL;   // slot 4*cl + m = member m of class cl
  constexpr int LD = CC + 1;
  extern __shared__ __align__(16) float2 sm3[];
  __shared__ double kr2s[CL];
  __shared__ int jlos[CL], jhis[CL], colof[CC];
  const int nk = v.nk;
  float2 *fin = sm3;                                 // [CC][nk]  source spectrum
  float2 *fout = fin + (size_t)CC * nk;              // [NZ][LD]  Stolt output / FFT work
  float2 *tw2 = fout + (size_t)NZ * LD;              // pass-2 twiddle rows
  const int tid = threadIdx.x;
  const int ncol = v.nx * v.ny;
  const int nclass = v.ncls;
  const int q0 = blockIdx.x * CL;
  const int f = blockIdx.y;
  if constexpr (DO_IFFT) sarfft2::build_tw2<NZ, (NZ == 512 ? 16 : 0), false>(tw2, v.tw_z, tid, K3C_NT);
  if (tid < CL) {
    const int q = q0 + tid;
    if (q < nclass) {
      const SarClass &c = v.cls[q];
      kr2s[tid] = c.kr2;
      jlos[tid] = c.jlo;
      jhis[tid] = c.jhi;
#pragma unroll
      for (int m = 0; m < 4; ++m) colof[4 * tid + m] = m < c.nmem ? c.col[m] : -1;
    } else {
      kr2s[tid] = 0.0;
      jlos[tid] = 0;
      jhis[tid] = -1;
#pragma unroll
      for (int m = 0; m < 4; ++m) colof[4 * tid + m] = -1;
    }
  }
  __syncthreads();
  // 1. member columns (streaming loads, 16 B per thread when n_k is even)
  const float2 *wf = v.w0 + (size_t)f * ncol * (size_t)nk;
  if ((nk & 1) == 0) {
    // 8 independent 16-byte loads in flight per thread before any store
    constexpr int U = 8;
    const int h2 = nk / 2, tot = CC * h2;
    for (int base = tid; base < tot; base += U * K3C_NT) {
      float4 t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * K3C_NT;
        const int sl = e / h2, i = e - sl * h2;
        t[u] = (e < tot && colof[sl] >= 0 && jhis[sl >> 2] >= jlos[sl >> 2])
                   ? __ldcs(reinterpret_cast<const float4 *>(wf + (size_t)colof[sl] * nk) + i)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * K3C_NT;
        const int sl = e / h2, i = e - sl * h2;
        if (e < tot) reinterpret_cast<float4 *>(fin + sl * nk)[i] = t[u];
      }
    }
  } else {
    for (int e = tid; e < CC * nk; e += K3C_NT) {
      const int sl = e / nk, i = e - sl * nk;
      if (colof[sl] >= 0 && jhis[sl >> 2] >= jlos[sl >> 2]) fin[e] = __ldcs(wf + (size_t)colof[sl] * nk + i);
    }
  }
  __syncthreads();
  // 2. Stolt pull over the in-band (class, j) pairs, filter at the two taps
  //    folded into the weights (readings R2-R5, R9)
  const double rr = v.rref[f + v.f0] * (1.0 / TWO_PI);
  int tot = 0;
#pragma unroll
  for (int cl = 0; cl < CL; ++cl) tot += jhis[cl] - jlos[cl] + 1;
  for (int idx = tid; idx < tot; idx += K3C_NT) {
    int cl = 0, j = idx;
#pragma unroll
    for (int q = 0; q < CL - 1; ++q) {
      const int len = jhis[cl] - jlos[cl] + 1;
      if (j >= len) {
        j -= len;
        ++cl;
      }
    }
    j += jlos[cl];
    const double kr2 = kr2s[cl];
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
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int sl = 4 * cl + m;
      if (colof[sl] < 0) break;
      float2 o = make_float2(0.f, 0.f);
      if (ok) o = cmac2(cmul2(wl, fin[sl * nk + i0]), wu, fin[sl * nk + i0 + 1]);
      fout[j * LD + sl] = o;
    }
  }
  __syncthreads();
  // 3. inverse z-FFT (out-of-band bins read as zero), columns stored [col][z]
  float2 *dst = v.w1 + (size_t)f * ncol * (size_t)NZ;
  auto load = [&](int c, int m) {
    const int cl = c >> 2;
    return (m >= jlos[cl] && m <= jhis[cl]) ? fout[m * LD + c] : make_float2(0.f, 0.f);
  };
  if constexpr (DO_IFFT) {
    sarfft2::fft_ctx<NZ, CC, LD, K3C_NT, +1, 0, true, (NZ == 512 ? 16 : 0), false, (NZ > 32)>(
        fout, NZ > 32 ? tw2 : v.tw_z, tid, load, [] {},
        [&](int c) {
          const int col = colof[c];
          return col >= 0 ? dst + (size_t)col * NZ : nullptr;
        },
        [&](float2 *p, int m, float2 x) {
          if (p) {
            SAR_IN(p + m, v.w1, v.w1_elems);
            st_mid(p + m, x);
          }
        });
  } else {
    for (int i = tid; i < CC * NZ; i += K3C_NT) {
      const int sl = i / NZ, z = i - sl * NZ;
      if (colof[sl] >= 0) dst[(size_t)colof[sl] * NZ + z] = load(sl, z);
    }
  }
}

// threads per consumer group, consumer groups (round-robin items), ring
// stages, mirror classes per item (compile-time overridable for A/B runs)
#ifndef K3P_G_
#define K3P_G_ 256
#endif
#ifndef K3P_NG_
#define K3P_NG_ 3
#endif
#ifndef K3P_S_
#define K3P_S_ 3
#endif
#ifndef K3P_CL_
#define K3P_CL_ 2
#endif
constexpr int K3P_G = K3P_G_;
constexpr int K3P_NG = K3P_NG_;
constexpr int K3P_S = K3P_S_;
constexpr int K3P_CL = K3P_CL_;
// group g takes items n = g (mod NG), which use stage n mod S: with NG | S
// every stage belongs to one group, so a group waiting on a stage's full
// barrier can never see the phase of another group's item (mbarrier parity
// waits cannot tell phases two apart)
static_assert(K3P_S % K3P_NG == 0, "K3 ring: the stage count must be a multiple of the group count");
// pass-2 split and row-major twiddle table of k3_pp's z-IFFT
template <int NZ, int CL>
struct K3PFft {
  static constexpr int R1S = NZ == 512 ? 16 : 0;
  static constexpr int R1 = R1S ? R1S : sarfft2::Split<NZ>::R1;
  // pass 2 split between thread pairs where C R1 butterflies would leave
  // half the group idle (N = 512 as 16 x 32, N = 256)
  static constexpr bool SPL = NZ / R1 >= 4 && 2 * (4 * CL) * R1 <= K3P_G;
  static constexpr int TWN = sarfft2::tw2_size<NZ, R1S, SPL>();
};
template <int NZ, int CL>
size_t k3pp_smem(int nk) {
  const size_t hdr = (sizeof(K3Hdr<CL>) + 15) & ~(size_t)15;
  return K3P_S * (hdr + (size_t)4 * CL * nk * sizeof(float2)) +
         K3P_NG * ((size_t)NZ * (4 * CL + 1)) * sizeof(float2) +
         ((size_t)NZ + nk) * sizeof(double) + (size_t)K3PFft<NZ, CL>::TWN * sizeof(float2);
}

template <int NZ, int CL, bool DO_IFFT>
__device__ __forceinline__ void k3pp_consume(const SarDeviceView &v, int nitems_f, int g, int gt,
                                             unsigned char *ring, size_t stage_bytes, size_t hdr_bytes,
                                             float2 *fout, const double *ks, const double *kzs, const float2 *tw,
                                             uint64_t *full, uint64_t *empty, int *colofs, int *slo, int *shi) {
  constexpr int CC = 4 * CL;
  constexpr int LD = CC + 1;
  const int nk = v.nk;
  const int ncol = v.nx * v.ny;
  const int nitems = nitems_f * v.F;
  unsigned n = g;
  for (int item = blockIdx.x + g * gridDim.x; item < nitems; item += K3P_NG * gridDim.x, n += K3P_NG) {
    const int st = n % K3P_S;
    sartma::mbar_wait(&full[st], (n / K3P_S) & 1);
    unsigned char *sb = ring + st * stage_bytes;
    const K3Hdr<CL> &h = *reinterpret_cast<const K3Hdr<CL> *>(sb);
    const float2 *fin = reinterpret_cast<const float2 *>(sb + hdr_bytes);
    const int f = h.f, nu = h.nused;
    const double rr = h.rr;
    // Stolt pull over the in-band (class, j) pairs only, the filter evaluated
    // at the two taps each pull uses and folded into the weights:
    //   O_j = (1-tau) H(k_i0) S_i0 + tau H(k_i0+1) S_i0+1
    int tot = 0;
#pragma unroll
    for (int cl = 0; cl < CL; ++cl) tot += h.jhi[cl] - h.jlo[cl] + 1;
    for (int idx = gt; idx < tot; idx += K3P_G) {
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
      const bool ok = stolt_pull(kzs[j], kr2, v.k0, v.inv_dk, v.dk, nk, v.stolt_delta, &i0, &tau);
      float2 wl = make_float2(0.f, 0.f), wu = wl;
      if (ok) {
        const float t = (float)tau;
        const float2 hl = filter_h(v, ks[i0], kr2, rr, i0);
        const float2 hu = filter_h(v, ks[i0 + 1], kr2, rr, i0 + 1);
        wl = make_float2((1.f - t) * hl.x, (1.f - t) * hl.y);
        wu = make_float2(t * hu.x, t * hu.y);
      }
      const int nm = h.nmem[cl];
      for (int m = 0; m < nm; ++m) {
        const int sl = h.mslot[cl][m];
        float2 o = make_float2(0.f, 0.f);
        if (ok) o = cmac2(cmul2(wl, fin[sl * nk + i0]), wu, fin[sl * nk + i0 + 1]);
        fout[j * LD + sl] = o;
      }
    }
    if (gt < CC) {
      const bool used = gt < nu;
      colofs[gt] = used ? h.colof[gt] : -1;
      slo[gt] = used ? h.jlo[h.clof[gt]] : NZ;
      shi[gt] = used ? h.jhi[h.clof[gt]] : -1;
    }
    sarfft2::sync<-1, K3P_G>(1 + g);
    if (gt == 0) sartma::mbar_arrive(&empty[st]);  // stage (header + columns) consumed
    // inverse z-FFT (out-of-band rows read as zero), columns stored contiguously
    float2 *dst = v.w1 + (size_t)f * ncol * (size_t)NZ;
    auto load = [&](int c, int m) {
      return (m >= slo[c] && m <= shi[c]) ? fout[m * LD + c] : make_float2(0.f, 0.f);
    };
    if (DO_IFFT) {
      // the output column's pointer is resolved once per butterfly, so every
      // store is one STG with an immediate offset
      using FT = K3PFft<NZ, CL>;
      sarfft2::fft_ctx<NZ, CC, LD, K3P_G, +1, -1, true, FT::R1S, FT::SPL, (NZ > 32)>(
          fout, tw, gt, load, [] {},
          [&](int c) {
            const int col = colofs[c];
            return col >= 0 ? dst + (size_t)col * NZ : nullptr;
          },
          [&](float2 *p, int m, float2 x) {
            if (p) {
            SAR_IN(p + m, v.w1, v.w1_elems);
            st_mid(p + m, x);
          }
          },
          1 + g);
    } else {
      for (int i = gt; i < CC * NZ; i += K3P_G) {
        const int sl = i / NZ, z = i - sl * NZ;
        if (sl < nu) dst[(size_t)colofs[sl] * NZ + z] = load(sl, z);
      }
    }
    sarfft2::sync<-1, K3P_G>(1 + g);  // fout / slot tables are rewritten by this group's next item
  }
}

template <int NZ, int CL, bool DO_IFFT>
__global__ void __launch_bounds__(K3P_NG * K3P_G + 32, 1) k3_pp(const SarDeviceView v, int nitems_f) {
  constexpr int CC = 4 * CL;
  constexpr int LD = CC + 1;
  constexpr int NTH = K3P_NG * K3P_G + 32;
  extern __shared__ __align__(16) unsigned char smp[];
  const int nk = v.nk;
  const size_t hdr_bytes = (sizeof(K3Hdr<CL>) + 15) & ~(size_t)15;
  const size_t stage_bytes = hdr_bytes + (size_t)CC * nk * sizeof(float2);
  unsigned char *ring = smp;
  float2 *grp = reinterpret_cast<float2 *>(smp + K3P_S * stage_bytes);
  const size_t grp_elems = (size_t)NZ * LD;                      // fout per group
  double *ks = reinterpret_cast<double *>(grp + K3P_NG * grp_elems);  // [nk]
  double *kzs = ks + nk;                                          // [NZ]
  float2 *tw = reinterpret_cast<float2 *>(kzs + NZ);              // pass-2 rows (K3PFft::TWN)
  __shared__ __align__(8) uint64_t full[K3P_S], empty[K3P_S];
  __shared__ int colofs[K3P_NG][CC], slo[K3P_NG][CC], shi[K3P_NG][CC];
  const int tid = threadIdx.x;
  for (int i = tid; i < nk; i += NTH) ks[i] = v.k[i];
  for (int i = tid; i < NZ; i += NTH) kzs[i] = v.kz[i];
  sarfft2::build_tw2<NZ, K3PFft<NZ, CL>::R1S, K3PFft<NZ, CL>::SPL>(tw, v.tw_z, tid, NTH);
  if (tid == 0) {
    for (int i = 0; i < K3P_S; ++i) {
      sartma::mbar_init(&full[i], 1);
      sartma::mbar_init(&empty[i], 1);
    }
    sartma::fence_barrier_init();
  }
  __syncthreads();
  const int ncol = v.nx * v.ny;
  const int nitems = nitems_f * v.F;
  if (tid >= K3P_NG * K3P_G) {
    // producer warp: lanes < CL read their class entry one item ahead,
    // write the stage header, and every member column is issued by its own
    // lane (cp.async.bulk, one mbarrier transaction per item)
    const int lane = tid & 31;
    const int nclass = v.ncls;
    auto fetch = [&](int item, SarClass &c) {
      const int f = item / nitems_f;
      const int q = (item - f * nitems_f) * CL + lane;
      if (item < nitems && lane < CL && q < nclass) {
        c = v.cls[q];
      } else {
        c.kr2 = 0.0;
        c.jlo = 0;
        c.jhi = -1;
        c.nmem = 0;
      }
    };
    SarClass cur, nxt;
    fetch(blockIdx.x, cur);
    unsigned n = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
      fetch(item + gridDim.x, nxt);   // in flight while this item is issued
      const int st = n % K3P_S;
      if (lane == 0 && n >= K3P_S) sartma::mbar_wait(&empty[st], ((n / K3P_S) - 1) & 1);
      __syncwarp();
      unsigned char *sb = ring + st * stage_bytes;
      K3Hdr<CL> &h = *reinterpret_cast<K3Hdr<CL> *>(sb);
      float2 *fin = reinterpret_cast<float2 *>(sb + hdr_bytes);
      const int f = item / nitems_f;
      // slot base of this lane's class = members of the classes before it
      const int mine = lane < CL ? cur.nmem : 0;
      int base = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, base, o);
        if (lane >= o) base += y;
      }
      const int cnt = __shfl_sync(0xffffffffu, base, CL - 1);
      base -= mine;
      if (lane < CL) {
        h.kr2[lane] = cur.kr2;
        h.jlo[lane] = cur.jlo;
        h.jhi[lane] = cur.jhi;
        h.nmem[lane] = cur.nmem;
        for (int m = 0; m < cur.nmem; ++m) {
          h.mslot[lane][m] = base + m;
          h.clof[base + m] = lane;
          h.colof[base + m] = cur.col[m];
        }
      }
      if (lane == 0) {
        h.nused = cnt;
        h.f = f;
        h.rr = v.rref[f + v.f0] * (1.0 / TWO_PI);
      }
      __syncwarp();
      // members of classes with no bin in band (jhi < jlo: zero output, kept
      // only to fill K4a's row boxes) are never read by the consumers: not loaded
      const bool ld = lane < cnt && h.jhi[h.clof[lane]] >= h.jlo[h.clof[lane]];
      const int nld = __popc(__ballot_sync(0xffffffffu, ld));
      if (lane == 0) sartma::mbar_arrive_expect_tx(&full[st], (uint32_t)nld * (uint32_t)nk * 8u);
      __syncwarp();
      const float2 *wf = v.w0 + (size_t)f * ncol * (size_t)nk;
      if (ld) {
        SAR_ASSERT(h.colof[lane] >= 0 && h.colof[lane] < ncol);
        SAR_IN(wf + (size_t)h.colof[lane] * nk + nk - 1, v.w0, v.w0_elems);
        sartma::bulk_g2s_stream<4>(fin + lane * nk, wf + (size_t)h.colof[lane] * nk, (uint32_t)nk * 8u, &full[st]);
      }
      cur = nxt;
    }
    return;
  }
  const int g = tid / K3P_G, gt = tid - g * K3P_G;
  k3pp_consume<NZ, CL, DO_IFFT>(v, nitems_f, g, gt, ring, stage_bytes, hdr_bytes, grp + g * grp_elems, ks, kzs, tw,
                                full, empty, colofs[g], slo[g], shi[g]);
}

// ------------------------------------------- K3, warp-specialised ----
// k3_ws (n_z = 512): the same arithmetic as k3_pp, split over three roles
// that run concurrently on every SM and hand work to each other through
// mbarriers only (no CTA-wide barrier on the data path):
//   * a producer warp fills an S-stage ring with the columns of the next
//     items (2 Stolt mirror classes = up to 8 columns, one cp.async.bulk per
//     column, as in k3_pp);
//   * KW_WS "Stolt" warps take every item: the bit-exact fp64 pull and the
//     filter at the two taps (readings R2-R5, R9), then the interpolated
//     in-band rows of each member column into one of KW_B column buffers
//     (out-of-band rows are masked later, never written); they hand the ring
//     stage back and the buffer on;
//   * 8 "FFT" warps, one per column slot of the buffer: each transforms its
//     column along z on its own (two-pass register FFT, 16 x 32, only
//     __syncwarp between the passes, pass 2 split over the lane halves) and
//     stores it to W1 [col][z] with 256-byte warp stores.
// A role waits only for the item it needs next, so the fp64 latency of the
// Stolt warps, the FFT warps' shared-memory round trips and the ring's
// transfer latency overlap instead of adding up behind barriers.
#ifndef KW_S_
#define KW_S_ 4
#endif
#ifndef KW_B_
#define KW_B_ 2
#endif
#ifndef KW_WS_
#define KW_WS_ 10
#endif
constexpr int KW_S = KW_S_;    // ring stages
constexpr int KW_B = KW_B_;    // column buffers
constexpr int KW_WS = KW_WS_;  // Stolt warps
#ifndef KW_FS_
#define KW_FS_ 1
#endif
constexpr int KW_WF = 8;    // FFT warps per set (= column slots of an item)
constexpr int KW_FS = KW_FS_;   // FFT warp sets; set s takes the items n = s (mod KW_FS)
constexpr int KW_CL = 2;    // mirror classes per item
#ifndef KW_ARR_
#define KW_ARR_ 32
#endif
constexpr int KW_ARR = KW_ARR_;
#ifndef KW_SLEEP
#define KW_SLEEP 1
#endif
#if KW_SLEEP
#define KW_WAIT sartma::mbar_wait_sleep
#else
#define KW_WAIT sartma::mbar_wait
#endif   // arrivals per warp on the hand-off barriers (1: lane 0 after __syncwarp)
constexpr int KW_NT = 32 * (1 + KW_WS + KW_WF * KW_FS);
// a buffer is always consumed by the same set (mbarrier parity waits cannot
// tell phases two apart)
static_assert(KW_B % KW_FS == 0, "k3_ws: the buffer count must be a multiple of the FFT set count");
template <int NZ>
struct KwGeom {
  static constexpr int R1 = 16, R2 = NZ / 16;         // pass 1 radix 16 (R2 = 32 butterflies)
  static constexpr int NZP = NZ + NZ / 16;             // padded column: m -> m + m/16
  static constexpr int TW2 = sarfft2::tw2_size<NZ, 16, true>();
  static constexpr size_t META = 128;                  // colof[8], slo[8], shi[8], f
  static constexpr size_t BUF = META + (size_t)KW_WF * NZP * sizeof(float2);
};
__device__ __forceinline__ int kw_pad(int m) { return m + (m >> 4); }

template <int NZ>
size_t k3ws_smem(int nk) {
  using G = KwGeom<NZ>;
  const size_t hdr = (sizeof(K3Hdr<KW_CL>) + 15) & ~(size_t)15;
  return KW_S * (hdr + (size_t)4 * KW_CL * nk * sizeof(float2)) + KW_B * G::BUF +
         ((size_t)NZ + nk) * sizeof(double) + (size_t)G::TW2 * sizeof(float2);
}

template <int NZ>
__global__ void __launch_bounds__(KW_NT, 1) k3_ws(const SarDeviceView v, int nitems_f) {
  using G = KwGeom<NZ>;
  constexpr int CL = KW_CL, CC = 4 * CL;
  static_assert(CC == KW_WF, "one FFT warp per column slot");
  static_assert(G::R2 == 32, "pass 1: one radix-16 butterfly per lane");
  extern __shared__ __align__(16) unsigned char smw[];
  const int nk = v.nk;
  const size_t hdr_bytes = (sizeof(K3Hdr<CL>) + 15) & ~(size_t)15;
  const size_t stage_bytes = hdr_bytes + (size_t)CC * nk * sizeof(float2);
  unsigned char *ring = smw;
  unsigned char *bufs = smw + KW_S * stage_bytes;
  double *ks = reinterpret_cast<double *>(bufs + KW_B * G::BUF);   // [nk]
  double *kzs = ks + nk;                                           // [NZ]
  float2 *tw = reinterpret_cast<float2 *>(kzs + NZ);               // pass-2 rows
  __shared__ __align__(8) uint64_t full[KW_S], empty[KW_S], full2[KW_B], empty2[KW_B];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < nk; i += KW_NT) ks[i] = v.k[i];
  for (int i = tid; i < NZ; i += KW_NT) kzs[i] = v.kz[i];
  sarfft2::build_tw2<NZ, 16, true>(tw, v.tw_z, tid, KW_NT);
  if (tid == 0) {
    for (int i = 0; i < KW_S; ++i) {
      sartma::mbar_init(&full[i], 1);
      sartma::mbar_init(&empty[i], KW_ARR * KW_WS);
    }
    for (int i = 0; i < KW_B; ++i) {
      sartma::mbar_init(&full2[i], KW_ARR * KW_WS);
      sartma::mbar_init(&empty2[i], KW_ARR * KW_WF);
    }
    sartma::fence_barrier_init();
  }
  __syncthreads();
  const int ncol = v.nx * v.ny;
  const int nitems = nitems_f * v.F;
  if (warp == 0) {
    // ---- producer: as k3_pp (class entries one item ahead, one bulk copy per member column)
    const int nclass = v.ncls;
    auto fetch = [&](int item, SarClass &c) {
      const int f = item / nitems_f;
      const int q = (item - f * nitems_f) * CL + lane;
      if (item < nitems && lane < CL && q < nclass) {
        c = v.cls[q];
      } else {
        c.kr2 = 0.0;
        c.jlo = 0;
        c.jhi = -1;
        c.nmem = 0;
      }
    };
    SarClass cur, nxt;
    fetch(blockIdx.x, cur);
    unsigned n = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
      fetch(item + gridDim.x, nxt);
      const int st = n % KW_S;
      if (lane == 0 && n >= KW_S) sartma::mbar_wait(&empty[st], ((n / KW_S) - 1) & 1);
      __syncwarp();
      unsigned char *sb = ring + st * stage_bytes;
      K3Hdr<CL> &h = *reinterpret_cast<K3Hdr<CL> *>(sb);
      float2 *fin = reinterpret_cast<float2 *>(sb + hdr_bytes);
      const int f = item / nitems_f;
      const int mine = lane < CL ? cur.nmem : 0;
      int base = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, base, o);
        if (lane >= o) base += y;
      }
      const int cnt = __shfl_sync(0xffffffffu, base, CL - 1);
      base -= mine;
      if (lane < CL) {
        h.kr2[lane] = cur.kr2;
        h.jlo[lane] = cur.jlo;
        h.jhi[lane] = cur.jhi;
        h.nmem[lane] = cur.nmem;
        for (int m = 0; m < cur.nmem; ++m) {
          h.mslot[lane][m] = base + m;
          h.clof[base + m] = lane;
          h.colof[base + m] = cur.col[m];
        }
      }
      if (lane == 0) {
        h.nused = cnt;
        h.f = f;
        h.rr = v.rref[f + v.f0] * (1.0 / TWO_PI);
      }
      __syncwarp();
      const bool ld = lane < cnt && h.jhi[h.clof[lane]] >= h.jlo[h.clof[lane]];
      const int nld = __popc(__ballot_sync(0xffffffffu, ld));
      if (lane == 0) sartma::mbar_arrive_expect_tx(&full[st], (uint32_t)nld * (uint32_t)nk * 8u);
      __syncwarp();
      const float2 *wf = v.w0 + (size_t)f * ncol * (size_t)nk;
      if (ld) {
        SAR_ASSERT(h.colof[lane] >= 0 && h.colof[lane] < ncol);
        SAR_IN(wf + (size_t)h.colof[lane] * nk + nk - 1, v.w0, v.w0_elems);
        sartma::bulk_g2s_stream<4>(fin + lane * nk, wf + (size_t)h.colof[lane] * nk, (uint32_t)nk * 8u, &full[st]);
      }
      cur = nxt;
    }
    return;
  }
  if (warp <= KW_WS) {
    // ---- Stolt warps: every item, (class, j) pairs strided over the KW_WS warps
    const int st_t = tid - 32;
    unsigned n = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
      const int st = n % KW_S, b = n % KW_B;
      KW_WAIT(&full[st], (n / KW_S) & 1);
      if (n >= KW_B) KW_WAIT(&empty2[b], ((n / KW_B) - 1) & 1);
      const unsigned char *sb = ring + st * stage_bytes;
      const K3Hdr<CL> &h = *reinterpret_cast<const K3Hdr<CL> *>(sb);
      const float2 *fin = reinterpret_cast<const float2 *>(sb + hdr_bytes);
      unsigned char *bb = bufs + b * G::BUF;
      int *meta = reinterpret_cast<int *>(bb);
      float2 *cols = reinterpret_cast<float2 *>(bb + G::META);
      const double rr = h.rr;
      int tot = 0;
#pragma unroll
      for (int cl = 0; cl < CL; ++cl) tot += h.jhi[cl] - h.jlo[cl] + 1;
      // an item has ~2 x 54 in-band pairs at Large (far fewer than Stolt
      // threads): the first pair goes to a thread that rotates by 3 warps per
      // item, so the fp64 chains of consecutive items run on different warps
      // (each warp runs ahead to the items it has work in)
      constexpr int NTS = 32 * KW_WS;
      const int rot = (int)((n * 96u) % (unsigned)NTS);
      const int t0 = st_t >= rot ? st_t - rot : st_t - rot + NTS;
      for (int idx = t0; idx < tot; idx += NTS) {
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
        const bool ok = stolt_pull(kzs[j], kr2, v.k0, v.inv_dk, v.dk, nk, v.stolt_delta, &i0, &tau);
        float2 wl = make_float2(0.f, 0.f), wu = wl;
        if (ok) {
          const float t = (float)tau;
          const float2 hl = filter_h(v, ks[i0], kr2, rr, i0);
          const float2 hu = filter_h(v, ks[i0 + 1], kr2, rr, i0 + 1);
          wl = make_float2((1.f - t) * hl.x, (1.f - t) * hl.y);
          wu = make_float2(t * hu.x, t * hu.y);
        }
        const int nm = h.nmem[cl];
        for (int m = 0; m < nm; ++m) {
          const int sl = h.mslot[cl][m];
          float2 o = make_float2(0.f, 0.f);
          if (ok) o = cmac2(cmul2(wl, fin[sl * nk + i0]), wu, fin[sl * nk + i0 + 1]);
          SAR_ASSERT(sl >= 0 && sl < KW_WF && j >= 0 && j < NZ);
          cols[sl * G::NZP + kw_pad(j)] = o;
        }
      }
      if (st_t < CC) {
        const bool used = st_t < h.nused;
        meta[st_t] = used ? h.colof[st_t] : -1;
        meta[CC + st_t] = used ? h.jlo[h.clof[st_t]] : NZ;
        meta[2 * CC + st_t] = used ? h.jhi[h.clof[st_t]] : -1;
      }
      if (st_t == 0) meta[3 * CC] = h.f;
      // every lane's stage reads were consumed by its stores above; arrive
      // (release) on both barriers, one arrival per warp after __syncwarp
      // (which orders the lanes' shared-memory writes before lane 0's release)
      if (KW_ARR == 1) __syncwarp();
      if (KW_ARR == 32 || lane == 0) {
        sartma::mbar_arrive(&empty[st]);
        sartma::mbar_arrive(&full2[b]);
      }
    }
    return;
  }
  // ---- FFT warps: warp w of set fs transforms column slot w of the set's items
  const int fw = warp - 1 - KW_WS, fs = fw / KW_WF, w = fw - fs * KW_WF;
  unsigned n = fs;
  for (int item = blockIdx.x + fs * gridDim.x; item < nitems; item += KW_FS * gridDim.x, n += KW_FS) {
    const int b = n % KW_B;
    KW_WAIT(&full2[b], (n / KW_B) & 1);
    unsigned char *bb = bufs + b * G::BUF;
    const int *meta = reinterpret_cast<const int *>(bb);
    float2 *col = reinterpret_cast<float2 *>(bb + G::META) + w * G::NZP;
    const int colof = meta[w], slo = meta[CC + w], shi = meta[2 * CC + w], f = meta[3 * CC];
    if (colof >= 0) {
      // pass 1: lane i, radix 16 over m = i + 32 r (rows outside [slo, shi] are zero)
      float2 x[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int m = lane + 32 * r;
        x[r] = (m >= slo && m <= shi) ? col[kw_pad(m)] : make_float2(0.f, 0.f);
      }
      __syncwarp();
      sarfft2::dft<16, +1>(x);
      sarfft2::static_for<0, 16>([&](auto P) {
        constexpr int p = decltype(P)::value;
        col[kw_pad(lane * 16 + sarfft2::freq_at(16, p))] = x[p];
      });
      __syncwarp();
      // pass 2, split over the lane halves (fft_ctx SPLIT2 with the row-major
      // twiddle table): ip = lane, i = ip mod 16
      constexpr int H = 16, TL = 32;
      const int ip = lane, i = ip & 15;
      float2 e = tw[H * TL + ip];
      e.y = -e.y;
      float2 g[H];
#pragma unroll
      for (int r = 0; r < H; ++r) {
        const float2 t = sarfft2::add(col[kw_pad(i + r * 16)], sarfft2::mul(col[kw_pad(i + (r + H) * 16)], e));
        if (r == 0) {
          g[0] = t;
        } else {
          float2 tw_ = tw[r * TL + ip];
          tw_.y = -tw_.y;
          g[r] = sarfft2::mul(t, tw_);
        }
      }
      sarfft2::dft<H, +1>(g);
      float2 *dst = v.w1 + ((size_t)f * ncol + colof) * (size_t)NZ;
      sarfft2::static_for<0, H>([&](auto P) {
        constexpr int p = decltype(P)::value;
        SAR_IN(dst + ip + 2 * sarfft2::freq_at(H, p) * 16, v.w1, v.w1_elems);
        st_mid(dst + ip + 2 * sarfft2::freq_at(H, p) * 16, g[p]);
      });
    }
    // the pass-2 reads of the buffer were consumed by the stores above
    if (KW_ARR == 1) __syncwarp();
    if (KW_ARR == 32 || lane == 0) sartma::mbar_arrive(&empty2[b]);
  }
}

// ------------------------------------------------- K3, NUFFT Stolt ----
// SAR_STOLT_NUFFT (reading R21): each filtered column is taken
// along z from its NON-uniform k_z,i = sqrt(4 k_i^2 - k_r^2) by a 1-D type-1
// NUFFT (fast Gaussian gridding, sigma = 2, W = 6) instead of the linear pull
// onto the uniform k_z grid + the z-IFFT.  One CTA per Stolt mirror class
// (the <= 4 columns sharing k_r^2, so the positions, the filter H and the
// Jacobian 4 k dk / (k_z dk_z) are computed once for the class):
//   1. member columns -> shared memory;
//   2. per sample i: in band iff 4 k_i^2 > k_r^2 and k_z,i >= k_z,0 (fp64, the
//      oracle's IEEE sequence), fine position sigma (k_z,i - k_z,0)/dk_z as
//      integer cell + fp32 fraction, weight H_i w_i;
//   3. gather onto the R = 2 n_z fine cells (periodic): cell l sums, in sample
//      order, weight_i F_i phi(l + kR - pos_i) over the contiguous sample
//      range with |l + kR - pos_i| <= W for every image k (positions increase
//      with i: binary search) -- deterministic, no atomics on the data;
//   4. inverse R-point FFT of the 4 fine columns (two-pass register FFT),
//      keep the n_z signed depths m, times 1/Phi(m) (host table), store
//      W1 [col][m mod n_z] (K4b applies 1/(nx ny nz)).
constexpr int K3N_NT = 256;
constexpr int K3N_W = 6;       // Gaussian half width (fine cells)
constexpr int K3N_LDW = 5;     // fine-grid row stride (4 members + pad)
template <int NZ>
size_t k3n_smem(int nk) {
  constexpr int R = 2 * NZ;
  return ((size_t)R * K3N_LDW + 5 * (size_t)nk) * sizeof(float2) + (size_t)nk * (sizeof(float) + sizeof(int)) +
         (size_t)(R + 4 * K3N_W + 8) * sizeof(int);
}

template <int NZ>
__global__ void __launch_bounds__(K3N_NT, 3) k3_nufft(const SarDeviceView v) {
  constexpr int R = 2 * NZ;
  constexpr int LDW = K3N_LDW;
  extern __shared__ __align__(16) float2 smn[];
  const int nk = v.nk;
  float2 *grid = smn;                                      // [R][LDW] fine cells x members
  float2 *fin = grid + (size_t)R * LDW;                    // [4][nk] member columns
  float2 *wgt = fin + (size_t)4 * nk;                      // [nk] H_i w_i
  float *posf = reinterpret_cast<float *>(wgt + nk);       // [nk] fraction of the fine position
  int *posb = reinterpret_cast<int *>(posf + nk);          // [nk] integer cell of the fine position
  int *cs = posb + nk;                                     // [<= R + 4W + 8] sample range starts
  __shared__ int colof[4], first;
  const int tid = threadIdx.x;
  const int q = blockIdx.x, f = blockIdx.y;
  const SarClass &c = v.cls[q];
  const int nm = c.nmem;
  const double kr2 = c.kr2;
  const int ncol = v.nx * v.ny;
  if (tid < 4) colof[tid] = tid < nm ? c.col[tid] : -1;
  if (tid == 0) first = nk;
  __syncthreads();
  const float2 *wf = v.w0 + (size_t)f * ncol * (size_t)nk;
  // 1-2. columns and per-sample terms (the fine grid starts at zero: cells
  //      no sample reaches are not written by the gather)
  for (int e = tid; e < R * LDW; e += K3N_NT) grid[e] = make_float2(0.f, 0.f);
  for (int e = tid; e < 4 * nk; e += K3N_NT) {
    const int m = e / nk, i = e - m * nk;
    fin[e] = colof[m] >= 0 ? __ldcs(wf + (size_t)colof[m] * nk + i) : make_float2(0.f, 0.f);
  }
  const double rr = v.rref[f + v.f0] * (1.0 / TWO_PI);
  const double kz0 = v.kz[0];
  const double inv_step = 1.0 / v.kz_step;
  for (int i = tid; i < nk; i += K3N_NT) {
    const double ki = v.k[i];
    const double qq = __dsub_rn(__dmul_rn(__dmul_rn(4.0, ki), ki), kr2);
    float2 w = make_float2(0.f, 0.f);
    int pb = 0;
    float pf = 0.f;
    if (qq > 0.0) {
      const double kz = __dsqrt_rn(qq);   // IEEE: the in-band decision is the oracle's
      if (kz >= kz0) {
        const double t = 2.0 * (kz - kz0) * inv_step;
        const double tb = floor(t);
        pb = (int)tb;
        pf = (float)(t - tb);
        // filter H = k_z e^{+j k_z R_ref} / P (reading R2), phase in turns
        double turns = kz * rr;
        turns -= rint(turns);
        float sn, cs;
        __sincosf((float)turns * 6.28318530717958647692f, &sn, &cs);
        // Jacobian 4 k dk / (k_z dk_z) times k_z of the filter: 4 k dk / dk_z
        const float amp = (float)(4.0 * ki * v.dk * inv_step);
        w = make_float2(amp * cs, amp * sn);
        if (v.pinv) w = cmul(w, v.pinv[i]);
        atomicMin(&first, i);
      }
    }
    wgt[i] = w;
    posb[i] = pb;
    posf[i] = pf;
  }
  __syncthreads();
  // 3. gather (in-band samples are the suffix [first, nk), positions
  //    increasing).  cs[j] = first sample with cell >= vlo + j - W - 1, so the
  //    samples within W of virtual cell lc are [cs[lc - vlo], cs[lc - vlo + 2W + 2]).
  //    Work item = (fine cell touched by some sample, quarter of its sample
  //    range): the touched cells are the circular range of the virtual cells
  //    [pos_min - W, pos_max + W] mod R; four consecutive lanes take the four
  //    quarters of one cell and sum all four members (positions, Gaussian and
  //    weights shared), then add their partial sums in a fixed shuffle order
  //    -- deterministic.  Every image p + kR of the cell is summed.
  const int i0 = first;
  const float inv2s2 = 0.5f / v.nu_s2;
  if (i0 < nk) {
    const int pmin = posb[i0], pmax = posb[nk - 1];
    const int vlo = pmin - K3N_W, vhi = pmax + 1 + K3N_W;
    const int nvc = vhi - vlo + 1;                      // virtual cells
    const int ncell = nvc < R ? nvc : R;                // physical cells touched
    const int ncs = nvc + 2 * K3N_W + 3;
    for (int j = tid; j < ncs; j += K3N_NT) {
      const int key = vlo + j - K3N_W - 1;
      int lo = i0, hi = nk;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (posb[mid] < key) lo = mid + 1;
        else hi = mid;
      }
      SAR_ASSERT(j < R + 4 * K3N_W + 8);
      cs[j] = lo;
    }
    __syncthreads();
    const int nit = (4 * ncell + 31) & ~31;   // whole warps (shuffles below)
    for (int it = tid; it < nit; it += K3N_NT) {
      const int qt = it & 3, jc = it >> 2;
      const bool live = jc < ncell;
      const int p = live ? ((vlo + jc) % R + R) % R : 0;
      float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      // images p + kR inside [vlo, vhi]: the first is vlo + ((p - vlo) mod R)
      for (int lc = live ? vlo + ((p - vlo) % R + R) % R : vhi + 1; lc <= vhi; lc += R) {
        const int j = lc - vlo;
        SAR_ASSERT(j >= 0 && j + 2 * K3N_W + 2 < ncs);
        const int lo = cs[j], n = cs[j + 2 * K3N_W + 2] - lo;
        const int a0 = lo + (n * qt) / 4, a1 = lo + (n * (qt + 1)) / 4;
        for (int i = a0; i < a1; ++i) {
          const float d = (float)(lc - posb[i]) - posf[i];
          if (fabsf(d) > (float)K3N_W) continue;
          const float ph = __expf(-d * d * inv2s2);
          const float2 wi = wgt[i];
          const float2 cw = make_float2(wi.x * ph, wi.y * ph);
#pragma unroll
          for (int m = 0; m < 4; ++m) acc[m] = cmac2(acc[m], cw, fin[m * nk + i]);
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        acc[m].x += __shfl_xor_sync(0xffffffffu, acc[m].x, 1);
        acc[m].y += __shfl_xor_sync(0xffffffffu, acc[m].y, 1);
        acc[m].x += __shfl_xor_sync(0xffffffffu, acc[m].x, 2);
        acc[m].y += __shfl_xor_sync(0xffffffffu, acc[m].y, 2);
      }
      if (live && qt == 0) {
        SAR_ASSERT(p >= 0 && p < R);
#pragma unroll
        for (int m = 0; m < 4; ++m) grid[p * LDW + m] = acc[m];
      }
    }
  }
  __syncthreads();
  // 4. inverse fine FFT, deconvolution, signed depths -> W1 [col][m mod nz]
  float2 *dst = v.w1 + (size_t)f * ncol * (size_t)NZ;
  sarfft2::fft_ctx<R, 4, LDW, K3N_NT, +1, 0, true>(
      grid, v.tw_z2, tid, [&](int cc, int n) { return grid[n * LDW + cc]; }, [] {},
      [&](int cc) {
        const int col = colof[cc];
        return col >= 0 ? dst + (size_t)col * NZ : nullptr;
      },
      [&](float2 *p, int n, float2 x) {
        if (p && (n < NZ / 2 || n >= R - NZ / 2)) {
          const int qz = n < NZ / 2 ? n : n - R + NZ;
          const float d = __ldg(v.sn_dec + qz);
          SAR_IN(p + qz, v.w1, v.w1_elems);
          st_mid(p + qz, make_float2(x.x * d, x.y * d));
        }
      });
}

// ------------------------------------------------------- K3, 2-D mode ----
// SAR_IMAGE_2D (reading R18): per Stolt mirror class (the <= 4 columns that
// share k_r^2), k_z,i = sqrt(4 k_i^2 - k_r^2) once, then for every plane s the
// back-propagation weights w_i = k_z,i exp(+j k_z,i (z_s - Z_0)) / P_i (phase
// in turns, fp64) and, per member column, the sum over k of S_i w_i (one warp
// per column: lanes stride over k, shuffle reduction).  Output W1[f][b][a][s]
// (planes fastest), which the y- and x-inverse kernels then transform like the
// z-chunks of the 3-D path.
constexpr int K3P2_NT = 256;   // 8 warps = 8 mirror classes per CTA
constexpr int K3P2_PS = 4;     // planes per pass (accumulators in registers)

__global__ void __launch_bounds__(K3P2_NT) k3_plane(const SarDeviceView v) {
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * (K3P2_NT / 32) + (threadIdx.x >> 5);
  const int f = blockIdx.y;
  const int nclass = v.ncls;
  if (q >= nclass) return;
  const SarClass &c = v.cls[q];
  const int nm = c.nmem, nk = v.nk, ns = v.nz;
  const int ncol = v.nx * v.ny;
  const double kr2 = c.kr2;
  const double zoff = v.rref[f + v.f0];   // z_s - Z_0 = (z_s - z_ref) + R_ref
  const float2 *wf = v.w0 + (size_t)f * ncol * (size_t)nk;
  const float2 *col[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) col[m] = wf + (size_t)(m < nm ? c.col[m] : c.col[0]) * nk;
  float2 *dst = v.w1 + (size_t)f * ncol * (size_t)ns;
  for (int s0 = 0; s0 < ns; s0 += K3P2_PS) {
    double tz[K3P2_PS];
#pragma unroll
    for (int u = 0; u < K3P2_PS; ++u) tz[u] = s0 + u < ns ? (__ldg(v.kz + s0 + u) + zoff) * (1.0 / TWO_PI) : 0.0;
    float2 acc[K3P2_PS][4];
#pragma unroll
    for (int u = 0; u < K3P2_PS; ++u)
#pragma unroll
      for (int m = 0; m < 4; ++m) acc[u][m] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int i = lane; i < nk; i += 32) {
      float2 x[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) x[m] = __ldcs(col[m] + i);
      const double ki = __ldg(v.k + i);
      const double qq = 4.0 * ki * ki - kr2;
      if (qq > 0.0) {
        const double kz = fast_dsqrt(qq);
        const float kzf = (float)kz;
        float2 pinv = make_float2(1.f, 0.f);
        if (v.pinv) pinv = v.pinv[i];
#pragma unroll
        for (int u = 0; u < K3P2_PS; ++u) {
          double turns = kz * tz[u];
          turns -= rint(turns);
          float sn, cs;
          __sincosf((float)turns * 6.28318530717958647692f, &sn, &cs);
          const float2 w = cmul(make_float2(kzf * cs, kzf * sn), pinv);
#pragma unroll
          for (int m = 0; m < 4; ++m) acc[u][m] = cmac2(acc[u][m], x[m], w);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < K3P2_PS; ++u)
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          acc[u][m].x += __shfl_xor_sync(0xffffffffu, acc[u][m].x, o);
          acc[u][m].y += __shfl_xor_sync(0xffffffffu, acc[u][m].y, o);
        }
    if (lane < 4 * K3P2_PS) {
      const int u = lane >> 2, m = lane & 3;
      float2 r = make_float2(0.f, 0.f);
#pragma unroll
      for (int uu = 0; uu < K3P2_PS; ++uu)
#pragma unroll
        for (int mm = 0; mm < 4; ++mm)
          if (uu == u && mm == m) r = acc[uu][mm];
      if (m < nm && s0 + u < ns) dst[(size_t)c.col[m] * ns + s0 + u] = r;
    }
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

template <typename K>
cudaError_t launch_v(K kernel, dim3 grid, int nt, size_t smem, cudaStream_t s, const SarDeviceView &v) {
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, nt, smem, s>>>(v);
  return cudaGetLastError();
}


}  // namespace

namespace {
// k3_pp with CL mirror classes per item if its shared memory fits
template <int N, int CL>
bool try_k3pp(const SarDeviceView &v, bool ifft, cudaStream_t s, int num_sms, cudaError_t *err) {
  const size_t smem = k3pp_smem<N, CL>(v.nk);
  if (smem > 225 * 1024) return false;
  const int nitems_f = (v.ncls + CL - 1) / CL;
  const int nitems = nitems_f * v.F;
  const int grid = nitems < num_sms ? nitems : num_sms;
  auto kern = ifft ? k3_pp<N, CL, true> : k3_pp<N, CL, false>;
  *err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (*err != cudaSuccess) return true;
  *err = launch_ex(kern, dim3(grid), dim3(K3P_NG * K3P_G + 32), smem, s, v, nitems_f);
  if (*err == cudaSuccess) *err = cudaGetLastError();
  return true;
}
}  // namespace

namespace {
}  // namespace

#ifndef K3_WS
#define K3_WS 1   // warp-specialised k3_ws at n_z = 512
#endif
cudaError_t launch_k3(const SarDeviceView &v, bool ifft, cudaStream_t s, int num_sms) {
  if (v.ncls == 0) return cudaSuccess;   // every column skipped (zero Stolt output)
  if (v.stolt_nufft) {
    if (!ifft) return cudaErrorInvalidValue;
    switch (v.nz) {
#define X(N)                                                                                           \
  case N: {                                                                                            \
    const size_t smem = k3n_smem<N>(v.nk);                                                             \
    if (smem > 227 * 1024) return cudaErrorInvalidValue;                                               \
    cudaError_t e = cudaFuncSetAttribute(k3_nufft<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                    \
    k3_nufft<N><<<dim3(v.ncls, v.F), K3N_NT, smem, s>>>(v);                                            \
    return cudaGetLastError();                                                                         \
  }
      X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512)
#undef X
    }
    return cudaErrorInvalidValue;
  }
  if (K3_WS && ifft && v.nz == 512 && (v.nk & 1) == 0 && !v.force_plain && k3ws_smem<512>(v.nk) <= 225 * 1024) {
    const size_t smem = k3ws_smem<512>(v.nk);
    const int nitems_f = (v.ncls + KW_CL - 1) / KW_CL;
    const int nitems = nitems_f * v.F;
    const int grid = nitems < num_sms ? nitems : num_sms;
    cudaError_t e = cudaFuncSetAttribute(k3_ws<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = launch_ex(k3_ws<512>, dim3(grid), dim3(KW_NT), smem, s, v, nitems_f);
    return e == cudaSuccess ? cudaGetLastError() : e;
  }
#ifndef K3PP_64
#define K3PP_64 0   // classes per item of k3_pp at n_z = 64 (0: k3_class there)
#endif
  if ((v.nk & 1) == 0 && (v.nz >= 128 || (K3PP_64 && v.nz == 64)) && !v.force_plain) {
    // n_z >= 256: 2 classes (<= 8 columns) per item; n_z = 128: 4 classes
    // (Freehand 0.065 -> 0.055 ms; at n_z = 64 k3_class stays faster:
    // Realtime 0.37 vs 0.43 ms with 8 classes per item)
    cudaError_t e = cudaSuccess;
    switch (v.nz) {
      case 64:
        if (try_k3pp<64, (K3PP_64 ? K3PP_64 : 4)>(v, ifft, s, num_sms, &e)) return e;
        break;
      case 128:
        if (try_k3pp<128, 4>(v, ifft, s, num_sms, &e)) return e;
        break;
      case 256:
        if (try_k3pp<256, K3P_CL>(v, ifft, s, num_sms, &e)) return e;
        break;
      case 512:
        if (try_k3pp<512, K3P_CL>(v, ifft, s, num_sms, &e)) return e;
        break;
      case 1024:
        if (try_k3pp<1024, K3P_CL>(v, ifft, s, num_sms, &e)) return e;
        break;
      default:
        break;
    }
  }
  const int nclass = v.ncls;
  switch (v.nz) {
#define X(N)                                                                                                   \
  case N: {                                                                                                    \
    constexpr int CLD = k3c_cl<N>();                                                                           \
    const bool big = k3c_smem<N, CLD>(v.nk) > 220 * 1024;                                                      \
    const int CL = big ? 1 : CLD;                                                                              \
    const size_t smem = big ? k3c_smem<N, 1>(v.nk) : k3c_smem<N, CLD>(v.nk);                                   \
    if (smem > 220 * 1024) return cudaErrorInvalidValue;                                                       \
    dim3 grid((nclass + CL - 1) / CL, v.F);                                                                    \
    auto kern = big ? (ifft ? k3_class<N, true, 1> : k3_class<N, false, 1>)                                   \
                    : (ifft ? k3_class<N, true, CLD> : k3_class<N, false, CLD>);                               \
    if (smem > 40 * 1024) {                                                                                    \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
      if (e != cudaSuccess) return e;                                                                          \
    }                                                                                                          \
    kern<<<grid, K3C_NT, smem, s>>>(v);                                                                        \
    return cudaGetLastError();                                                                                 \
  }
    SAR_SIZES(X)
#undef X
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_k3_plane(const SarDeviceView &v, cudaStream_t s) {
  const int nclass = v.ncls;
  if (nclass == 0) return cudaSuccess;
  const int cpb = K3P2_NT / 32;
  k3_plane<<<dim3((nclass + cpb - 1) / cpb, v.F), K3P2_NT, 0, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_stolt_index(const SarDeviceView &v, const int32_t *cols, int n, int32_t *i0, float *tau,
                               cudaStream_t s) {
  const long long total = (long long)n * v.nz;
  if (total == 0) return cudaSuccess;
  const int nt = 256;
  k_stolt_index<<<(unsigned)((total + nt - 1) / nt), nt, 0, s>>>(v, cols, n, i0, tau);
  return cudaGetLastError();
}


}  // namespace sark
