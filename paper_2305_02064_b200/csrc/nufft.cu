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

// K1s on the tensor cores (k1s_tc).  For one block of 4 x 4 fine cells, one
// frame and 64 wavenumbers the spread is a real GEMM
//     D[m][c] = sum_e A[m][e] B[e][c],   m = 2 k + (re, im),  c = cell,
// with A[m][e] the rotated sample s_e(k) e^{+j k beta_e} of entry e (its real or
// imaginary part) and B[e][c] = phi(j_x - U_e) phi(j_y - V_e) its Gaussian
// weight (reading R19).  tcgen05.mma kind::tf32, M = 128, N = 16, K = 8 per
// instruction, the fp32 product kept by splitting both operands into TF32
// hi + lo parts (3xTF32: hi.hi + hi.lo + lo.hi; the dropped lo.lo term is
// ~2^-22 relative).  The accumulator lives in TMEM (16 of 32 allocated
// columns).  The entries are taken 32 at a time: the 256 threads stage the
// chunk's operands (each thread: 8 entries of one wavenumber, coalesced loads
// along k, the rotation as in K1s, hi/lo split, 16-byte stores into the
// canonical no-swizzle K-major layout) into one of two buffers while the MMAs
// of the previous chunk run; one thread issues the 12 MMAs of a chunk and
// commits them to the buffer's mbarrier.  Epilogue: warps 0-3 read the
// accumulator rows (tcgen05.ld 32x32b), pair re/im by a shuffle and store the
// 16 cells' 64 wavenumbers into the fine grid.  Deterministic (fixed order).
namespace tc {
constexpr int KCH = 64;          // wavenumbers per CTA (M = 2 * KCH = 128)
constexpr int EC = 32;           // entries per chunk (4 MMAs of K = 8)
constexpr int NT = 256;
constexpr int ASBO = 1088;       // byte stride between 8-row core groups of A (1024 + 64: conflict-free stores)
constexpr int ABYTES = 16 * ASBO;                 // one A part (128 rows)
constexpr int BBYTES = 2 * (EC / 4) * 128;        // one B part (16 rows)
constexpr int BUF = 2 * ABYTES + 2 * BBYTES;      // one stage: A hi, A lo, B hi, B lo
#ifndef TC_STAGES
#define TC_STAGES 4
#endif
constexpr int S = TC_STAGES;
constexpr int SMEM = S * BUF;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// TF32 part of x by truncation (one LOP3): the tensor core reads the top 19
// bits of an fp32 operand, so hi = trunc(x) and lo = x - hi (exact in fp32,
// |lo| < 2^-10 |x|, itself truncated by the hardware: the split keeps ~2^-20)
__device__ __forceinline__ float tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
// shared-memory matrix descriptor: K-major, no swizzle, version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}
// instruction descriptor: D f32, A/B tf32, K-major, M x N
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ bool try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
}  // namespace tc

// Warp-specialised: 8 builder warps (warp w stages entries 4w .. 4w+3 of a
// chunk, all 64 wavenumbers and their 16 weights) + 1 MMA warp, on an S-stage
// mbarrier ring (full: 8 warp arrivals; empty: the MMA commit); no CTA-wide
// barrier in the loop.
__global__ void __launch_bounds__(tc::NT + 32, 1) k1s_tc(const __grid_constant__ SarDeviceView v,
                                                         const float2 *__restrict__ s) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smt[];
  __shared__ __align__(8) uint64_t full[S], empty[S], done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = v.nk;
  const int nkc = (nk + KCH - 1) / KCH;
  const int bx = blockIdx.x, by = blockIdx.y;
  const int f = blockIdx.z / nkc, kc = blockIdx.z - f * nkc;
  const int blk = (f * v.sp_nby + by) * v.sp_nbx + bx;
  const int e0 = v.sp_off[blk], e1 = v.sp_off[blk + 1];
  const int nchunks = (e1 - e0 + EC - 1) / EC;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[i])), "r"(NT / 32));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (warp == NT / 32) {
    // ---- MMA warp: one lane issues the 12 MMAs of every chunk ----
    if (lane == 0) {
      for (int c = 0; c < nchunks; ++c) {
        const int st = c % S;
        while (!try_wait(&full[st], (c / S) & 1)) {
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(smt + st * BUF), b0 = a0 + 2 * ABYTES;
#pragma unroll
        for (int q = 0; q < EC / 8; ++q) {
          const uint64_t dah = sdesc(a0 + q * 256, 128, ASBO), dal = sdesc(a0 + ABYTES + q * 256, 128, ASBO);
          const uint64_t dbh = sdesc(b0 + q * 256, 128, (EC / 4) * 128);
          const uint64_t dbl = sdesc(b0 + BBYTES + q * 256, 128, (EC / 4) * 128);
#ifndef TC_NO_MMA
          mma(tmem, dah, dbh, (c | q) != 0);
          mma(tmem, dah, dbl, 1);
          mma(tmem, dal, dbh, 1);
#else
          if (c == 0 && q == 0) mma(tmem, dah, dbh, 0);
#endif
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&empty[st])));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&done)));
    }
  } else {
    // ---- builder warps: entries 4 warp .. 4 warp + 3 of every chunk ----
    const bool rot = !v.no_comp;
    const float W = (float)v.nu_w, inv2s2 = 0.5f / v.nu_s2;
    const int k0 = kc * KCH + lane, k1 = k0 + 32;   // this lane's two wavenumbers
    const float kt0 = v.kturn[k0 < nk ? k0 : nk - 1], kt1 = v.kturn[k1 < nk ? k1 : nk - 1];
    // the samples of a chunk are loaded one chunk ahead (memory-level
    // parallelism across chunks: each warp walks its chunks in order)
    // entry records are loaded two chunks ahead, the samples one chunk ahead
    // (memory-level parallelism across chunks: each warp walks its chunks in order)
    auto fetch_ent = [&](int c) {
      const int eb = e0 + c * EC + 4 * warp;
      float4 q = make_float4(__int_as_float(0), 0.f, 0.f, 0.f);
      if (c < nchunks && lane < 4 && eb + lane < e1) {
        const SarSpreadEntry E = v.sp_ent[eb + lane];
        q = make_float4(__int_as_float(E.row), E.du, E.dv, E.beta);
      }
      return q;
    };
    auto fetch = [&](int c, const float4 &q, float2 (&y0)[4], float2 (&y1)[4]) {
      const int ebase = e0 + c * EC + 4 * warp;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = __shfl_sync(0xffffffffu, __float_as_int(q.x), u);
        const bool lv = c < nchunks && ebase + u < e1;
        y0[u] = (lv && k0 < nk) ? __ldg(s + (size_t)row * nk + k0) : make_float2(0.f, 0.f);
        y1[u] = (lv && k1 < nk) ? __ldg(s + (size_t)row * nk + k1) : make_float2(0.f, 0.f);
      }
    };
    float4 qn = fetch_ent(0), qn2 = fetch_ent(1);
    float2 xn0[4], xn1[4];
    fetch(0, qn, xn0, xn1);
    for (int c = 0; c < nchunks; ++c) {
      const int st = c % S;
      const int ebase = e0 + c * EC + 4 * warp;
      const float4 q = qn;
      float2 x0[4], x1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = xn0[u];
        x1[u] = xn1[u];
      }
      qn = qn2;
      qn2 = fetch_ent(c + 2);
      fetch(c + 1, qn, xn0, xn1);
      if (c >= S)
        while (!try_wait(&empty[st], ((c / S) - 1) & 1)) {
        }
      unsigned char *bb = smt + st * BUF;
      float du[4], dv[4];
      bool live[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        du[u] = __shfl_sync(0xffffffffu, q.y, u);
        dv[u] = __shfl_sync(0xffffffffu, q.z, u);
        const float beta = __shfl_sync(0xffffffffu, q.w, u);
        live[u] = ebase + u < e1;
        if (rot) {
          float t0 = beta * kt0, t1 = beta * kt1;
          t0 -= (t0 + 12582912.f) - 12582912.f;
          t1 -= (t1 + 12582912.f) - 12582912.f;
          float s0, c0, s1, c1;
          __sincosf(t0 * 6.28318530717958647692f, &s0, &c0);
          __sincosf(t1 * 6.28318530717958647692f, &s1, &c1);
          x0[u] = cmul(x0[u], make_float2(c0, s0));
          x1[u] = cmul(x1[u], make_float2(c1, s1));
        }
      }
      // A: rows 2k (re) and 2k+1 (im), this warp's 16-byte piece (core column ki = warp)
      unsigned char *ah = bb, *al = bb + ABYTES;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 *x = h ? x1 : x0;
        const int m0 = 2 * (lane + 32 * h);
        const float4 hr = make_float4(tf32(x[0].x), tf32(x[1].x), tf32(x[2].x), tf32(x[3].x));
        const float4 hi_ = make_float4(tf32(x[0].y), tf32(x[1].y), tf32(x[2].y), tf32(x[3].y));
        const float4 lr = make_float4(x[0].x - hr.x, x[1].x - hr.y, x[2].x - hr.z, x[3].x - hr.w);
        const float4 li = make_float4(x[0].y - hi_.x, x[1].y - hi_.y, x[2].y - hi_.z, x[3].y - hi_.w);
        const int off = (m0 >> 3) * ASBO + warp * 128 + (m0 & 7) * 16;
        *reinterpret_cast<float4 *>(ah + off) = hr;
        *reinterpret_cast<float4 *>(ah + off + 16) = hi_;
        *reinterpret_cast<float4 *>(al + off) = lr;
        *reinterpret_cast<float4 *>(al + off + 16) = li;
      }
      // B: the 4 entries' weights on the 16 cells (lanes 0-15: cell = lane; one 16-byte piece per cell row)
      if (lane < 16) {
        const int cell = lane, cy = cell / SAR_SP_BX, cx = cell - cy * SAR_SP_BX;
        float w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float dx = (float)cx - du[u], dy = (float)cy - dv[u];
          w[u] = (live[u] && fabsf(dx) <= W && fabsf(dy) <= W) ? __expf(-dy * dy * inv2s2) * __expf(-dx * dx * inv2s2)
                                                               : 0.f;
        }
        const float4 wh = make_float4(tf32(w[0]), tf32(w[1]), tf32(w[2]), tf32(w[3]));
        const float4 wl = make_float4(w[0] - wh.x, w[1] - wh.y, w[2] - wh.z, w[3] - wh.w);
        const int off = ((cell >> 3) * (EC / 4) + warp) * 128 + (cell & 7) * 16;
        *reinterpret_cast<float4 *>(bb + 2 * ABYTES + off) = wh;
        *reinterpret_cast<float4 *>(bb + 2 * ABYTES + BBYTES + off) = wl;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[st])) : "memory");
    }
    // ---- epilogue: warps 0-3 read the accumulator rows ----
    if (warp < 4) {
      if (nchunks > 0)
        while (!try_wait(&done, 0)) {
        }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int m = warp * 32 + lane;
      const int ko = kc * KCH + (m >> 1);
      const int RX = 2 * v.nx, RY = 2 * v.ny;
      float2 *dst = v.wh + ((size_t)(f * RY + by * SAR_SP_BY) * RX + bx * SAR_SP_BX) * (size_t)nk + ko;
#pragma unroll
      for (int cell = 0; cell < 16; ++cell) {
        const float mine = nchunks > 0 ? __uint_as_float(r[cell]) : 0.f;
        const float other = __shfl_xor_sync(0xffffffffu, mine, 1);
        const int cy = cell / SAR_SP_BX, cx = cell - cy * SAR_SP_BX;
        if (!(lane & 1) && ko < nk) __stcs(dst + ((size_t)cy * RX + cx) * nk, make_float2(mine, other));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
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
#ifdef SAR_TC_SPREAD   // experiment: slower than the FP32 gather
  if (!v.force_plain) {
    const int nkc = (v.nk + tc::KCH - 1) / tc::KCH;
    dim3 grid(v.sp_nbx, v.sp_nby, v.F * nkc);
    cudaError_t e = cudaFuncSetAttribute(k1s_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM);
    if (e != cudaSuccess) return e;
    k1s_tc<<<grid, tc::NT + 32, tc::SMEM, s>>>(v, data);
    return cudaGetLastError();
  }
#endif
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
