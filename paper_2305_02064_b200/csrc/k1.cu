// k1.cu -- K1: correction + MIMO accumulation + x-FFT (Eqs. (11)-(12), P:183-193;
// reading R6), raw samples -> W0.  The launcher picks the TMA-pipelined
// persistent kernel when the geometry allows, else the plain one.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <type_traits>
#include <vector>

#include "common.cuh"

#ifndef K1_GROUPS
#define K1_GROUPS 2
#endif

namespace sark {
namespace {

// ---------------------------------------------------------------- K1 ------
// One CTA = (k chunk, virtual row vy, frame f).  Thread item e covers
// (vx, kk) = (item / 16, item % 16).  For pair (t,r) the pose row feeding vy
// is iy = (vy - j^y_tr) mod ny (reading R6); it contributes iff iy < npy and
// ix = (vx - j^x_tr) mod nx < npx.  Rotation phase in turns:
// k_i beta / (2 pi) = kturn_i * (apose_p + bpair_tr), reduced to [-1/2, 1/2]
// before the SFU sincos (|k beta| reaches tens of radians).
template <int NX, bool DO_FFT>
__global__ void __launch_bounds__(nt_for(NX), minb_for(NX))
    k1_correct_xfft(const SarDeviceView v, const float2 *__restrict__ s) {
  constexpr int NT = nt_for(NX);
  constexpr int ITEMS = NX * KC;
  constexpr int E = (ITEMS + NT - 1) / NT;
  extern __shared__ float2 tile[];  // [NX][16]
  const int tid = threadIdx.x;
  const int kbase = blockIdx.x * KC;
  const int vy = v.vy0 + blockIdx.y;
  const int f = blockIdx.z;

  static_assert(NT % KC == 0, "k lane of a thread is fixed: kk = tid % 16");
  float2 acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = make_float2(0.f, 0.f);
  const float kt = kbase + (tid & (KC - 1)) < v.nk ? __ldg(v.kturn + kbase + (tid & (KC - 1))) : 0.f;

  for (int pr = 0; pr < v.npair; ++pr) {
    int iy = vy - v.jy[pr];
    if (iy < 0) iy += v.ny;
    if (iy >= v.npy) continue;  // uniform over the CTA
    const int t = pr / v.nr, r = pr - t * v.nr;
    const size_t rowbase = ((size_t)((f + v.f0) * v.nt + t) * v.nr + r) * (size_t)v.P + (size_t)iy * v.npx;
    const float2 *srow = s + rowbase * (size_t)v.nk;
    const float *ap = v.apose + (size_t)(f + v.f0) * v.P + (size_t)iy * v.npx;
    const float bp = v.bpair[(f + v.f0) * v.npair + pr];
    const int jx = v.jx[pr];
    // issue a batch of EB independent loads before consuming any (memory-level
    // parallelism without holding all E samples in registers)
    constexpr int EB = E < 8 ? E : 8;
#pragma unroll
    for (int e0 = 0; e0 < E; e0 += EB) {
      float2 val[EB];
      float bet[EB];
#pragma unroll
      for (int u = 0; u < EB; ++u) {
        const int item = tid + (e0 + u) * NT;
        const int kk = item & (KC - 1);
        const int vx = item >> 4;
        int ix = vx - jx;
        if (ix < 0) ix += NX;
        const bool ok = (ITEMS % NT == 0 || item < ITEMS) && ix < v.npx && kbase + kk < v.nk;
        val[u] = ok ? __ldcs(srow + (size_t)ix * v.nk + (kbase + kk)) : make_float2(0.f, 0.f);
        bet[u] = ok ? __ldg(ap + ix) : 0.f;
      }
      if (v.no_comp) {
#pragma unroll
        for (int u = 0; u < EB; ++u) acc[e0 + u] = cadd(acc[e0 + u], val[u]);
      } else {
#pragma unroll
        for (int u = 0; u < EB; ++u) {
          float turns = (bet[u] + bp) * kt;
          turns -= rintf(turns);
          float sn, cs;
          __sincosf(turns * 6.28318530717958647692f, &sn, &cs);
          acc[e0 + u] = cadd(acc[e0 + u], cmul(val[u], make_float2(cs, sn)));
        }
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

  float2 *out = v.w0 + ((size_t)(f * v.nvy + blockIdx.y) * NX) * (size_t)v.nk;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int kk = item & (KC - 1), vx = item >> 4;
    const int k = kbase + kk;
    if (k < v.nk) {
      if (v.slab_lg >= 0) {   // slab stage 1: packed per destination rank (or into the peer)
        const int h = vx >> v.slab_lg, al = vx & ((1 << v.slab_lg) - 1);
        v.slab_dst[h][(((size_t)blockIdx.y << v.slab_lg) + al) * v.nk + k] = tile[item];
      } else {
        SAR_IN(out + (size_t)vx * v.nk + k, v.w0, v.w0_elems);
        out[(size_t)vx * v.nk + k] = tile[item];
      }
    }
  }
}

// SAR_GRID_NEAREST (reading R20): K1 with the plan's node lists instead of
// the raster rows.  One CTA = (k chunk, lattice row vy, frame f), thread item
// (vx, kk) as in k1_correct_xfft; item (vx, kk) sums, in list order, every
// (pair, pose) sample row the plan put on node (f, vy, vx), rotated by
// exp(+j k beta) with beta = -2 d_z + beta_MIMO (Eqs. (11)-(12)); then the same
// x-FFT and store.  With every pose on its raster node the lists hold one
// row per pair in pair order, so the result equals k1_correct_xfft's bit for
// bit (same rotation code, same order).
template <int NX, bool DO_FFT>
__global__ void __launch_bounds__(nt_for(NX), minb_for(NX))
    k1_nearest(const SarDeviceView v, const float2 *__restrict__ s) {
  constexpr int NT = nt_for(NX);
  constexpr int ITEMS = NX * KC;
  constexpr int E = (ITEMS + NT - 1) / NT;
  extern __shared__ float2 tile[];  // [NX][16]
  const int tid = threadIdx.x;
  const int kbase = blockIdx.x * KC;
  const int vy = blockIdx.y;
  const int f = blockIdx.z;
  static_assert(NT % KC == 0, "k lane of a thread is fixed: kk = tid % 16");
  const int k = kbase + (tid & (KC - 1));
  const float kt = k < v.nk ? __ldg(v.kturn + k) : 0.f;
  const int *off = v.nn_off + ((size_t)(f + v.f0) * v.ny + vy) * NX;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int vx = item >> 4;
    float2 acc = make_float2(0.f, 0.f);
    if (k < v.nk) {
      const int q1 = __ldg(off + vx + 1);
      // up to 4 entries' samples in flight, summed in list order
      for (int q = __ldg(off + vx); q < q1; q += 4) {
        SarNearEntry en[4];
        float2 val[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          en[u] = q + u < q1 ? v.nn_ent[q + u] : SarNearEntry{0, 0.f};
          SAR_ASSERT(en[u].row >= 0 && (size_t)en[u].row < v.raw_rows);
          val[u] = q + u < q1 ? __ldcs(s + (size_t)en[u].row * v.nk + k) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (q + u >= q1) break;
          if (v.no_comp) {
            acc = cadd(acc, val[u]);
          } else {
            float turns = en[u].beta * kt;
            turns -= rintf(turns);
            float sn, cs;
            __sincosf(turns * 6.28318530717958647692f, &sn, &cs);
            acc = cadd(acc, cmul(val[u], make_float2(cs, sn)));
          }
        }
      }
    }
    tile[item] = acc;  // tile[vx*16 + kk]
  }
  __syncthreads();
  if constexpr (DO_FFT) sarfft::tile_fft<NX, KC, KC, NT, -1>(tile, v.tw_x, tid);
  float2 *out = v.w0 + ((size_t)(f * v.nvy + vy) * NX) * (size_t)v.nk;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int kk = item & (KC - 1), vx = item >> 4;
    if (kbase + kk < v.nk) {
      SAR_IN(out + (size_t)vx * v.nk + kbase + kk, v.w0, v.w0_elems);
      out[(size_t)vx * v.nk + kbase + kk] = tile[item];
    }
  }
}

// Persistent, TMA-pipelined K1 (used when n_k is even, npx % 4 == 0 and the
// step phasor below is accurate).  One CTA (1024 threads) per SM walks a flat
// sequence of "jobs" = (work item (frame, vy, k chunk of K1C), valid pair, box
// of up to br pose rows).  Thread 0 keeps K1_STAGES jobs in flight: one 2-D
// TMA box of raw samples [br poses][K1C k] (32 KB) plus the matching [br]
// slice of the -2 d_z table, completing on the stage's mbarrier.  The chunk
// width K1C = 8192/NX keeps the [NX][K1C] x-FFT tile at 64 KB.
// Each thread owns one pose row of the box and 4 consecutive k: the rotation
// exp(j k_i beta) of the first comes from the SFU (phase reduced in turns),
// the next three from multiplying by the step exp(j dk beta), evaluated as its
// 5th-order Taylor polynomial (|dk beta| <= 0.25 is checked by the plan, so
// the truncation error is < 4e-7).  Complex arithmetic uses the sm_100 paired
// fp32 instructions (__ffma2_rn / __fmul2_rn).
// REGACC (all j^x offsets 0, e.g. a linear Tx/Rx column along y): each thread
// always owns the same (vx, k) elements, so sums stay in registers; otherwise
// they accumulate in the shared tile (one owner per element per job).
struct K1Job {
  int item, pr, b;
};

__device__ __forceinline__ bool k1_pair_valid(const SarDeviceView &v, int vy, int pr) {
  int iy = vy - v.jy[pr];
  if (iy < 0) iy += v.ny;
  return iy < v.npy;
}

// advance j to the next job of this CTA (item stride = gridDim.x); false at the end
__device__ __forceinline__ bool k1_next(const SarDeviceView &v, K1Job &j, int nitems, int nchunk, int nbox) {
  if (++j.b < nbox) return true;
  j.b = 0;
  for (;;) {
    const int vy = v.vy0 + (j.item / nchunk) % v.nvy;
    while (++j.pr < v.npair)
      if (k1_pair_valid(v, vy, j.pr)) return true;
    j.item += gridDim.x;
    j.pr = -1;
    if (j.item >= nitems) return false;
  }
}

// NG = 2 (REGACC with two boxes per pose row): the consumer warps form two
// groups, group g takes the jobs of box g (every other job, its own two ring
// stages), so the halves of a row advance independently instead of every
// stage waiting for all 16 warps.
template <int NX, bool REGACC, bool SLAB, int NG>
__global__ void __launch_bounds__(K1_NT + 32, 1)
    k1_correct_xfft_tma(const SarDeviceView v, const __grid_constant__ CUtensorMap tm_s,
                        const __grid_constant__ CUtensorMap tm_ap, int br, int nbox, int nitems) {
  constexpr int C = k1c_for(NX);
  constexpr int BRMAX = K1_BOX_BYTES / (C * 8);
  constexpr int TPR = C / K1_KT;                 // consumer threads per box row
  constexpr int GT = K1_NT / NG;                 // consumer threads per group
  constexpr int RPP = GT / TPR;                  // box rows per consumer pass
  constexpr int UPB = BRMAX / RPP;               // box rows per consumer thread
  constexpr int MAXB = NX / BRMAX > 0 ? NX / BRMAX : 1;  // boxes per pose row (<= 2)
  constexpr int NB = NG == 2 ? 1 : MAXB;         // boxes a thread accumulates
  static_assert(NG == 1 || (REGACC && MAXB == 2 && K1_STAGES % 2 == 0), "two groups: REGACC, two boxes");
  constexpr int NWARP = K1_NT / 32 / NG;         // arrivals per stage
  extern __shared__ __align__(128) unsigned char smraw[];
  float2 *tile = reinterpret_cast<float2 *>(smraw);                       // [NX][C]
  unsigned char *stages = smraw + (size_t)NX * C * sizeof(float2);
  constexpr size_t STAGE = K1_BOX_BYTES + BRMAX * sizeof(float);
  float2 *tws = reinterpret_cast<float2 *>(stages + K1_STAGES * STAGE);   // [NX] twiddles
  __shared__ __align__(8) uint64_t full[K1_STAGES], empty[K1_STAGES];
  const int tid = threadIdx.x;
  const int nchunk = (v.nk + C - 1) / C;
  if (tid == 0) {
    for (int i = 0; i < K1_STAGES; ++i) {
      sartma::mbar_init(&full[i], 1);
      sartma::mbar_init(&empty[i], NWARP);
    }
    sartma::fence_barrier_init();
  }
  if (!REGACC)
    for (int i = tid; i < NX * C; i += K1_NT + 32) tile[i] = make_float2(0.f, 0.f);
  for (int i = tid; i < NX; i += K1_NT + 32) tws[i] = v.tw_x[i];
  __syncthreads();

  if (tid >= K1_NT) {
    // ---------------- producer warp: one elected lane issues every TMA ----------------
    if (tid == K1_NT) {
      const uint32_t tx_bytes = (uint32_t)(br * C * sizeof(float2) + br * sizeof(float));
      K1Job j{(int)blockIdx.x, -1, nbox - 1};
      if (j.item < nitems) {
        unsigned n = 0;
        for (bool more = k1_next(v, j, nitems, nchunk, nbox); more; more = k1_next(v, j, nitems, nchunk, nbox), ++n) {
          const int st = n % K1_STAGES;
          if (n >= K1_STAGES) sartma::mbar_wait(&empty[st], ((n / K1_STAGES) - 1) & 1);
          const int kc = j.item % nchunk, rest = j.item / nchunk;
          const int vy = v.vy0 + rest % v.nvy, f = rest / v.nvy;
          int iy = vy - v.jy[j.pr];
          if (iy < 0) iy += v.ny;
          const int t = j.pr / v.nr, r = j.pr - t * v.nr;
          const long long row =
              ((long long)((f + v.f0) * v.nt + t) * v.nr + r) * v.P + (long long)iy * v.npx + j.b * br;
          unsigned char *sb = stages + st * STAGE;
          sartma::mbar_arrive_expect_tx(&full[st], tx_bytes);
          sartma::tma_load_2d_stream<1>(sb, &tm_s, kc * C, (int)row, &full[st]);
          sartma::tma_load_2d(sb + K1_BOX_BYTES, &tm_ap, j.b * br, (f + v.f0) * v.npy + iy, &full[st]);
        }
      }
    }
    return;
  }

  // ---------------- consumers: 512 threads ----------------
  const int g = NG == 2 ? tid / GT : 0;        // group: the box it accumulates (NG = 2)
  const int gtid = tid - g * GT;
  const int kq = (gtid % TPR) * K1_KT;  // first of this thread's K1_KT k within the chunk
  const int r0 = gtid / TPR;           // first of this thread's box rows
  const int lane = tid & 31;
  const float dkt = (float)(v.dk);
  unsigned jobctr = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int kc = item % nchunk, rest = item / nchunk;
    const int vyl = rest % v.nvy, f = rest / v.nvy;
    const int vy = v.vy0 + vyl;
    const int k0 = kc * C + kq;
    const float kt = k0 < v.nk ? __ldg(v.kturn + k0) : 0.f;
    float2 acc[REGACC ? NB * UPB * K1_KT : 1];
#pragma unroll
    for (int u = 0; u < (REGACC ? NB * UPB * K1_KT : 1); ++u) acc[u] = make_float2(0.f, 0.f);
    for (int pr = 0; pr < v.npair; ++pr) {
      if (!k1_pair_valid(v, vy, pr)) continue;
      const float bp = v.bpair[(f + v.f0) * v.npair + pr];
      const int jx = v.jx[pr];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        if (b >= nbox) break;
        const int st = jobctr % K1_STAGES;
        const unsigned ph = (jobctr / K1_STAGES) & 1;
        ++jobctr;
        if (NG == 2 && b != g) continue;   // the other group's job
        sartma::mbar_wait(&full[st], ph);
        const float2 *sv = reinterpret_cast<const float2 *>(stages + st * STAGE);
        const float *sap = reinterpret_cast<const float *>(stages + st * STAGE + K1_BOX_BYTES);
        // the warp's rows of the box go to registers and the stage is handed
        // back before the rotation, so the producer refills it meanwhile
        constexpr int NV = K1_KT / 2;   // float4 (2 samples) per row and thread
        float4 rv[UPB][NV];
        float rbeta[UPB];
#pragma unroll
        for (int w = 0; w < UPB; ++w) {
          const int il = r0 + w * RPP;
          const int ix = b * br + il;
#pragma unroll
          for (int q = 0; q < NV; ++q) rv[w][q] = make_float4(0.f, 0.f, 0.f, 0.f);
          rbeta[w] = 0.f;
          if (il < br && ix < v.npx) {
#pragma unroll
            for (int q = 0; q < NV; ++q) rv[w][q] = *reinterpret_cast<const float4 *>(sv + il * C + kq + 2 * q);
            rbeta[w] = sap[il];
          }
        }
        // the stage is refilled by TMA (async proxy) after this warp's arrival:
        // the proxy fence makes the shared-memory reads above complete first
        sartma::fence_proxy_async();
        __syncwarp();
        if (lane == 0) sartma::mbar_arrive(&empty[st]);
#pragma unroll
        for (int w = 0; w < UPB; ++w) {
          const int il = r0 + w * RPP;
          const int ix = b * br + il;
          if (il < br && ix < v.npx) {
            float2 val[K1_KT];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
              val[2 * q] = make_float2(rv[w][q].x, rv[w][q].y);
              val[2 * q + 1] = make_float2(rv[w][q].z, rv[w][q].w);
            }
            if (!v.no_comp) {
              const float beta = rbeta[w] + bp;
              float turns = beta * kt;
              turns -= rintf(turns);
              float2 rot;
              __sincosf(turns * 6.28318530717958647692f, &rot.y, &rot.x);
              const float x = dkt * beta, x2 = x * x;
              const float2 step = make_float2(fmaf(x2, fmaf(x2, 1.f / 24.f, -0.5f), 1.f),
                                              x * fmaf(x2, fmaf(x2, 1.f / 120.f, -1.f / 6.f), 1.f));
#pragma unroll
              for (int u = 0; u < K1_KT; ++u) {
                val[u] = cmul2(val[u], rot);
                if (u + 1 < K1_KT) rot = cmul2(rot, step);
              }
            }
            if constexpr (REGACC) {
#pragma unroll
              for (int u = 0; u < K1_KT; ++u)
                acc[((NG == 2 ? 0 : b) * UPB + w) * K1_KT + u] =
                    __fadd2_rn(acc[((NG == 2 ? 0 : b) * UPB + w) * K1_KT + u], val[u]);
            } else {
              int vx = ix + jx;
              if (vx >= NX) vx -= NX;
              float2 *t = tile + vx * C + kq;
#pragma unroll
              for (int u = 0; u < K1_KT; ++u) t[u] = __fadd2_rn(t[u], val[u]);
            }
          }
        }
        if (!REGACC) sarfft::tile_sync<1, K1_NT>();  // tile updates of this job complete
      }
    }
    if constexpr (REGACC) {
      // vx = ix for every pair: scatter the register sums into the tile
#pragma unroll
      for (int bb = 0; bb < NB; ++bb)
#pragma unroll
        for (int w = 0; w < UPB; ++w) {
          const int b = NG == 2 ? g : bb;
          const int il = r0 + w * RPP;
          const int ix = b * br + il;
          if (b < nbox && il < br && ix < NX)
#pragma unroll
            for (int u = 0; u < K1_KT; ++u) tile[ix * C + kq + u] = acc[(bb * UPB + w) * K1_KT + u];
        }
      // rows not covered by any box (npx < NX) are zero
      for (int i = nbox * br * C + tid; i < NX * C; i += K1_NT) tile[i] = make_float2(0.f, 0.f);
    }
    sarfft::tile_sync<1, K1_NT>();
    // x-FFT (two-pass register FFT; the accumulation tile doubles as its work
    // tile) with the transformed rows stored straight to W0
    float2 *out = v.w0 + ((size_t)(f * v.nvy + vyl) * NX) * (size_t)v.nk + kc * C;
    const int cmax = v.nk - kc * C;
    sarfft2::fft<NX, C, C, K1_NT, -1, 1, false, (NX == 512 ? 16 : 0)>(
        tile, tws, tid, [&](int c, int m) { return tile[m * C + c]; }, [] {},
        [&](int c, int m, float2 x) {
          if (c < cmax) {
            if constexpr (SLAB) {   // slab stage 1: packed per destination rank (or into the peer)
              const int h = m >> v.slab_lg, al = m & ((1 << v.slab_lg) - 1);
              __stcs(v.slab_dst[h] + (((size_t)vyl << v.slab_lg) + al) * v.nk + kc * C + c, x);
            } else {
              SAR_IN(out + (size_t)m * v.nk + c, v.w0, v.w0_elems);
              st_mid(out + (size_t)m * v.nk + c, x);
            }
          }
        });
    sarfft::tile_sync<1, K1_NT>();
    if (!REGACC) {
      for (int i = tid; i < NX * C; i += K1_NT) tile[i] = make_float2(0.f, 0.f);
      sarfft::tile_sync<1, K1_NT>();
    }
  }
}

template <typename K>
cudaError_t launch(K kernel, dim3 grid, int nt, size_t smem, cudaStream_t s, const SarDeviceView &v,
                   const float2 *arg) {
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, nt, smem, s>>>(v, arg);
  return cudaGetLastError();
}


}  // namespace

cudaError_t launch_k1(const SarDeviceView &v, const float2 *data, bool fft, cudaStream_t s,
                      const CUtensorMap *tm_s, const CUtensorMap *tm_ap, int br, bool regacc, int num_sms) {
  if (v.nearest) {
    dim3 grid((v.nk + KC - 1) / KC, v.ny, v.F);
    const size_t smem = (size_t)v.nx * KC * sizeof(float2);
    switch (v.nx) {
#define X(N)                                                                                   \
  case N:                                                                                      \
    return fft ? launch(k1_nearest<N, true>, grid, nt_for(N), smem, s, v, data)               \
               : launch(k1_nearest<N, false>, grid, nt_for(N), smem, s, v, data);
      SAR_SIZES(X)
#undef X
    }
    return cudaErrorInvalidValue;
  }
  if (fft && tm_s && tm_ap && v.nx >= 64 && v.nx <= 512 && v.k1_step_ok) {
    const int C = k1c_for(v.nx);
    const int nchunk = (v.nk + C - 1) / C;
    const int nitems = nchunk * v.nvy * v.F;
    const int nbox = (v.npx + br - 1) / br;
    const int brmax = K1_BOX_BYTES / (C * 8);
    const size_t smem = (size_t)v.nx * C * sizeof(float2) + K1_STAGES * ((size_t)K1_BOX_BYTES + brmax * sizeof(float)) +
                        (size_t)v.nx * sizeof(float2);
    const int grid = nitems < num_sms ? nitems : num_sms;
    switch (v.nx) {
#define X(N)                                                                                          \
  case N: {                                                                                           \
    auto kern = v.slab_lg >= 0 ? (regacc ? k1_correct_xfft_tma<N, true, true, 1> : k1_correct_xfft_tma<N, false, true, 1>) \
                               : (regacc ? k1_correct_xfft_tma<N, true, false, 1> : k1_correct_xfft_tma<N, false, false, 1>); \
    if (K1_GROUPS == 2 && (N == 512 || N == 128) && regacc && nbox == 2 && v.slab_lg < 0)            \
      kern = k1_correct_xfft_tma<N, true, false, ((N == 512 || N == 128) && K1_GROUPS == 2) ? 2 : 1>; \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                   \
    e = launch_ex(kern, dim3(grid), dim3(K1_NT + 32), smem, s, v, *tm_s, *tm_ap, br, nbox, nitems);       \
    if (e != cudaSuccess) return e;                                                                   \
    return cudaGetLastError();                                                                        \
  }
      X(64) X(128) X(256) X(512)
#undef X
    }
  }
  dim3 grid((v.nk + KC - 1) / KC, v.nvy, v.F);
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


}  // namespace sark
