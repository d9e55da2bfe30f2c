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

#include <stdlib.h>
#include <string>
#include <type_traits>
#include <vector>

#include "fft_tile.cuh"
#include "fft_reg.cuh"
#include "tma.cuh"
#include "plan_internal.h"

using sarfft::cadd;
using sarfft::cmul;

namespace {

constexpr int KC = 16;  // k (or z) chunk: 16 complex64 = one 128-byte line
constexpr double TWO_PI = 6.283185307179586476925286766559;
constexpr double BAND_EPS = 1e-9;  // reading R9

constexpr int nt_for(int n) { return n <= 32 ? 32 : (n < 512 ? n : 512); }
// resident CTAs requested per SM: 1024 threads' worth (caps registers at 64 per
// thread) except for the 1024-point tiles, whose 32 elements per thread need more
constexpr int minb_for(int n) { return n >= 1024 ? 1 : 1024 / nt_for(n); }
// persistent tile kernels: 2N threads (8 elements each of a 16-column tile),
// capped at 1024, and as many CTAs per SM as make 1024 threads
constexpr int ntp_for(int n) { return 2 * n < 64 ? 64 : (2 * n > 1024 ? 1024 : 2 * n); }
constexpr int ctas_for(int n) { return 1024 / ntp_for(n); }

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
  const int vy = blockIdx.y;
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
    const size_t rowbase = ((size_t)(f * v.nt + t) * v.nr + r) * (size_t)v.P + (size_t)iy * v.npx;
    const float2 *srow = s + rowbase * (size_t)v.nk;
    const float *ap = v.apose + (size_t)f * v.P + (size_t)iy * v.npx;
    const float bp = v.bpair[f * v.npair + pr];
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
constexpr int K1_STAGES = 4;
constexpr int K1_BOX_BYTES = 32768;
constexpr int K1_NT = 512;   // consumer threads (+1 producer warp)
constexpr int K1_KT = 4;  // consecutive k per thread

constexpr int k1c_for(int nx) { return nx >= 512 ? 16 : (nx == 256 ? 32 : 64); }

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
    const int vy = (j.item / nchunk) % v.ny;
    while (++j.pr < v.npair)
      if (k1_pair_valid(v, vy, j.pr)) return true;
    j.item += gridDim.x;
    j.pr = -1;
    if (j.item >= nitems) return false;
  }
}

// acc += a * b (complex), two paired-fp32 FMAs
__device__ __forceinline__ float2 cmac2(float2 acc, float2 a, float2 b) {
  acc = __ffma2_rn(make_float2(a.x, a.x), b, acc);
  return __ffma2_rn(make_float2(-a.y, a.y), make_float2(b.y, b.x), acc);
}
__device__ __forceinline__ float2 cmul2(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(-a.y, a.y), make_float2(b.y, b.x)));
}

template <int NX, bool REGACC>
__global__ void __launch_bounds__(K1_NT + 32, 1)
    k1_correct_xfft_tma(const SarDeviceView v, const __grid_constant__ CUtensorMap tm_s,
                        const __grid_constant__ CUtensorMap tm_ap, int br, int nbox, int nitems) {
  constexpr int C = k1c_for(NX);
  constexpr int BRMAX = K1_BOX_BYTES / (C * 8);
  constexpr int TPR = C / K1_KT;                 // consumer threads per box row
  constexpr int RPP = K1_NT / TPR;               // box rows per consumer pass
  constexpr int UPB = BRMAX / RPP;               // box rows per consumer thread
  constexpr int MAXB = NX / BRMAX > 0 ? NX / BRMAX : 1;  // boxes per pose row (<= 2)
  constexpr int NWARP = K1_NT / 32;
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
          const int vy = rest % v.ny, f = rest / v.ny;
          int iy = vy - v.jy[j.pr];
          if (iy < 0) iy += v.ny;
          const int t = j.pr / v.nr, r = j.pr - t * v.nr;
          const long long row = ((long long)(f * v.nt + t) * v.nr + r) * v.P + (long long)iy * v.npx + j.b * br;
          unsigned char *sb = stages + st * STAGE;
          sartma::mbar_arrive_expect_tx(&full[st], tx_bytes);
          sartma::tma_load_2d(sb, &tm_s, kc * C, (int)row, &full[st]);
          sartma::tma_load_2d(sb + K1_BOX_BYTES, &tm_ap, j.b * br, f * v.npy + iy, &full[st]);
        }
      }
    }
    return;
  }

  // ---------------- consumers: 512 threads ----------------
  const int kq = (tid % TPR) * K1_KT;   // first of this thread's 4 k within the chunk
  const int r0 = tid / TPR;            // first of this thread's box rows
  const int lane = tid & 31, warp = tid >> 5;
  const float dkt = (float)(v.dk);
  unsigned jobctr = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int kc = item % nchunk, rest = item / nchunk;
    const int vy = rest % v.ny, f = rest / v.ny;
    const int k0 = kc * C + kq;
    const float kt = k0 < v.nk ? __ldg(v.kturn + k0) : 0.f;
    float2 acc[REGACC ? MAXB * UPB * K1_KT : 1];
#pragma unroll
    for (int u = 0; u < (REGACC ? MAXB * UPB * K1_KT : 1); ++u) acc[u] = make_float2(0.f, 0.f);
    for (int pr = 0; pr < v.npair; ++pr) {
      if (!k1_pair_valid(v, vy, pr)) continue;
      const float bp = v.bpair[f * v.npair + pr];
      const int jx = v.jx[pr];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        if (b >= nbox) break;
        const int st = jobctr % K1_STAGES;
        sartma::mbar_wait(&full[st], (jobctr / K1_STAGES) & 1);
        ++jobctr;
        const float2 *sv = reinterpret_cast<const float2 *>(stages + st * STAGE);
        const float *sap = reinterpret_cast<const float *>(stages + st * STAGE + K1_BOX_BYTES);
#pragma unroll
        for (int w = 0; w < UPB; ++w) {
          const int il = r0 + w * RPP;
          const int ix = b * br + il;
          if (il < br && ix < v.npx) {
            const float4 v01 = *reinterpret_cast<const float4 *>(sv + il * C + kq);
            const float4 v23 = *reinterpret_cast<const float4 *>(sv + il * C + kq + 2);
            float2 val[4] = {make_float2(v01.x, v01.y), make_float2(v01.z, v01.w), make_float2(v23.x, v23.y),
                             make_float2(v23.z, v23.w)};
            if (!v.no_comp) {
              const float beta = sap[il] + bp;
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
                acc[(b * UPB + w) * K1_KT + u] = __fadd2_rn(acc[(b * UPB + w) * K1_KT + u], val[u]);
            } else {
              int vx = ix + jx;
              if (vx >= NX) vx -= NX;
              float2 *t = tile + vx * C + kq;
#pragma unroll
              for (int u = 0; u < K1_KT; ++u) t[u] = __fadd2_rn(t[u], val[u]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) sartma::mbar_arrive(&empty[st]);
        if (!REGACC) sarfft::tile_sync<1, K1_NT>();  // tile updates of this job complete
      }
    }
    if constexpr (REGACC) {
      // vx = ix for every pair: scatter the register sums into the tile
#pragma unroll
      for (int b = 0; b < MAXB; ++b)
#pragma unroll
        for (int w = 0; w < UPB; ++w) {
          const int il = r0 + w * RPP;
          const int ix = b * br + il;
          if (b < nbox && il < br && ix < NX)
#pragma unroll
            for (int u = 0; u < K1_KT; ++u) tile[ix * C + kq + u] = acc[(b * UPB + w) * K1_KT + u];
        }
      // rows not covered by any box (npx < NX) are zero
      for (int i = nbox * br * C + tid; i < NX * C; i += K1_NT) tile[i] = make_float2(0.f, 0.f);
    }
    sarfft::tile_sync<1, K1_NT>();
    // x-FFT (two-pass register FFT; the accumulation tile doubles as its work
    // tile) with the transformed rows stored straight to W0
    float2 *out = v.w0 + ((size_t)(f * v.ny + vy) * NX) * (size_t)v.nk + kc * C;
    const int cmax = v.nk - kc * C;
    sarfft2::fft<NX, C, C, K1_NT, -1, 1, false, (NX == 512 ? 16 : 0)>(
        tile, tws, tid, [&](int c, int m) { return tile[m * C + c]; }, [] {},
        [&](int c, int m, float2 x) {
          if (c < cmax) __stcs(out + (size_t)m * v.nk + c, x);
        });
    sarfft::tile_sync<1, K1_NT>();
    if (!REGACC) {
      for (int i = tid; i < NX * C; i += K1_NT) tile[i] = make_float2(0.f, 0.f);
      sarfft::tile_sync<1, K1_NT>();
    }
  }
}

// ------------------------------------------------------------ K2 / K4a ----
// FFT along the middle (y) axis of a [F][N][nx][inner] complex volume for one
// (chunk of 16 along `inner`, column a, frame f).
template <int N, int DIR>
__global__ void __launch_bounds__(nt_for(N), minb_for(N))
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

// Persistent, TMA-pipelined variant of k_fft_mid (used when `inner` is even,
// i.e. the rows are 16-byte aligned).  One CTA per SM loops over work items
// (chunk, column a, frame); the [N][16] tile of item i+1 is in flight
// (cp.async.bulk.tensor, mbarrier completion) while item i is transformed,
// and finished tiles go back with TMA stores, so the SM's load queue never
// drains between tiles.  Box = {16 inner elements, 1 column, <=256 rows}.
template <int N, int DIR>
__global__ void __launch_bounds__(ntp_for(N), ctas_for(N))
    k_fft_mid_tma(const __grid_constant__ CUtensorMap tm, const float2 *__restrict__ twg, int nx, int nchunk,
                  int nitems) {
  constexpr int NT = ntp_for(N);
  constexpr int ROWS = N < 256 ? N : 256;
  constexpr int NBOX = N / ROWS;
  constexpr uint32_t TILE_BYTES = N * KC * sizeof(float2);
  extern __shared__ __align__(128) float2 smt[];  // [2][N][16]
  __shared__ __align__(8) uint64_t full[2];
  __shared__ float2 tw[N];
  const int tid = threadIdx.x;
  for (int i = tid; i < N; i += NT) tw[i] = twg[i];
  if (tid == 0) {
    sartma::mbar_init(&full[0], 1);
    sartma::mbar_init(&full[1], 1);
    sartma::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int item, int st) {
    const int chunk = item % nchunk, rest = item / nchunk;
    const int a = rest % nx, f = rest / nx;
    sartma::mbar_arrive_expect_tx(&full[st], TILE_BYTES);
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx)
      sartma::tma_load_3d(smt + (size_t)st * N * KC + bx * ROWS * KC, &tm, chunk * KC, a, f * N + bx * ROWS,
                          &full[st]);
  };
  int item = blockIdx.x;
  if (tid == 0 && item < nitems) issue(item, 0);
  for (int it = 0; item < nitems; ++it, item += gridDim.x) {
    const int st = it & 1;
    const int next = item + gridDim.x;
    if (tid == 0 && next < nitems) {
      sartma::bulk_wait_read0();  // the store of stage st^1 has left shared memory
      issue(next, st ^ 1);
    }
    sartma::mbar_wait(&full[st], (it >> 1) & 1);
    float2 *tile = smt + (size_t)st * N * KC;
    sarfft::tile_fft<N, KC, KC, NT, DIR>(tile, tw, tid);
    sartma::fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      const int chunk = item % nchunk, rest = item / nchunk;
      const int a = rest % nx, f = rest / nx;
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx)
        sartma::tma_store_3d(&tm, chunk * KC, a, f * N + bx * ROWS, tile + bx * ROWS * KC);
      sartma::bulk_commit();
    }
  }
  if (tid == 0) sartma::bulk_wait0();
}

// Warp-specialised persistent mid-axis FFT (K2 / K4a, ny <= 512, `inner`
// even).  A producer warp streams [N][16] tiles (3-D TMA boxes {16 inner, 1
// column, <=256 rows}) into an S-stage mbarrier ring; NTC consumer threads run
// the two-pass register FFT (fft_reg.cuh), hand the stage back right after
// the pass-1 loads, and store the transformed rows straight to global memory
// (each warp store = two full 128-byte lines).
template <int N>
constexpr int mid2_stages() { return N >= 256 ? 2 : 4; }
template <int N>
constexpr size_t mid2_smem() {
  return ((size_t)mid2_stages<N>() * N * KC + (size_t)N * KC + N) * sizeof(float2);
}
template <int N>
constexpr int mid2_ctas() {
  return (int)((200 * 1024) / mid2_smem<N>()) < 1 ? 1 : (int)((200 * 1024) / mid2_smem<N>());
}

template <int N, int DIR>
__global__ void __launch_bounds__(sarfft2::nt_fft<N, KC>() + 32)
    k_fft_mid2(const __grid_constant__ CUtensorMap tm, float2 *__restrict__ data, const float2 *__restrict__ twg,
               int nx, int inner, int nchunk, int nitems) {
  constexpr int NTC = sarfft2::nt_fft<N, KC>();
  constexpr int S = mid2_stages<N>();
  constexpr int ROWS = N < 256 ? N : 256;
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
        sartma::mbar_arrive_expect_tx(&full[st], TILE_BYTES);
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx)
          sartma::tma_load_3d(ring + (size_t)st * N * KC + bx * ROWS * KC, &tm, chunk * KC, a, f * N + bx * ROWS,
                              &full[st]);
      }
    }
    return;
  }
  const size_t row = (size_t)nx * inner;
  unsigned n = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
    const int st = n % S;
    sartma::mbar_wait(&full[st], (n / S) & 1);
    const int chunk = item % nchunk, rest = item / nchunk;
    const int a = rest % nx, f = rest / nx;
    const float2 *stage = ring + (size_t)st * N * KC;
    float2 *base = data + ((size_t)f * N * nx + a) * (size_t)inner + chunk * KC;
    const int cmax = inner - chunk * KC;
    sarfft2::fft<N, KC, KC, NTC, DIR, 1, false>(
        work, tw, tid, [&](int c, int m) { return stage[m * KC + c]; },
        [&] {
          if (tid == 0) sartma::mbar_arrive(&empty[st]);
        },
        [&](int c, int m, float2 v) {
          if (c < cmax) __stcs(base + (size_t)m * row + c, v);
        });
  }
}

// Warp-specialised persistent K4b (nx <= 512, n_z even): [nx][16 z] tiles of
// W1 row y stream through an S-stage TMA ring; the consumers run the inverse
// x-FFT (pass 2 mapped so that one warp owns 32 consecutive x of one z) and
// write |o|/(nx ny nz) (or the scaled complex value) straight into the rolled
// image rows (reading R8, R11): coalesced 128-byte segments, no transpose
// buffer.
template <int NX, bool CPLX>
constexpr size_t k4b2_smem() {
  return ((size_t)2 * NX * KC + (size_t)NX * (KC + 1) + NX) * sizeof(float2);
}
template <int NX>
constexpr int k4b2_ctas() {
  return (int)((200 * 1024) / k4b2_smem<NX, false>()) < 1 ? 1 : (int)((200 * 1024) / k4b2_smem<NX, false>());
}

template <int NX, bool CPLX>
__global__ void __launch_bounds__(sarfft2::nt_fft<NX, KC>() + 32)
    k4_xifft_mag2(const SarDeviceView v, const __grid_constant__ CUtensorMap tm, void *__restrict__ img, int nzc,
                  int nitems) {
  constexpr int NTC = sarfft2::nt_fft<NX, KC>();
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
  for (int i = tid; i < NX; i += NTC + 32) tw[i] = v.tw_x[i];
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
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx)
          sartma::tma_load_3d(ring + (size_t)st * NX * KC + bx * ROWS * KC, &tm, zc * KC, bx * ROWS, fy, &full[st]);
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
    OT *outp = reinterpret_cast<OT *>(img) + ((size_t)f * nz * v.ny + iy) * NX;
    const float2 *stage = ring + (size_t)st * NX * KC;
    sarfft2::fft<NX, KC, KC + 1, NTC, +1, 1, true>(
        work, tw, tid, [&](int c, int m) { return stage[m * KC + c]; },
        [&] {
          if (tid == 0) sartma::mbar_arrive(&empty[st]);
        },
        [&](int c, int a, float2 o) {
          const int z = zc * KC + c;
          if (z < nz) {
            int m = z + v.zroll;
            if (m >= nz) m -= nz;
            const int ix = (a - rx) & (NX - 1);
            if constexpr (CPLX) {
              __stcs(reinterpret_cast<float2 *>(outp) + (size_t)m * zstride + ix, make_float2(o.x * sc, o.y * sc));
            } else {
              __stcs(reinterpret_cast<float *>(outp) + (size_t)m * zstride + ix, sqrtf(fmaf(o.x, o.x, o.y * o.y)) * sc);
            }
          }
        });
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
template <int NZ>
size_t k3c_smem(int nk) {
  constexpr int CL = k3c_cl<NZ>();
  return ((size_t)4 * CL * nk + (size_t)NZ * (4 * CL + 1)) * sizeof(float2);
}

template <int NZ, bool DO_IFFT>
__global__ void __launch_bounds__(K3C_NT, 4) k3_class(const SarDeviceView v) {
  constexpr int CL = k3c_cl<NZ>();
  constexpr int CC = 4 * CL;   // slot 4*cl + m = member m of class cl
  constexpr int LD = CC + 1;
  extern __shared__ __align__(16) float2 sm3[];
  __shared__ double kr2s[CL];
  __shared__ int jlos[CL], jhis[CL], colof[CC];
  const int nk = v.nk;
  float2 *fin = sm3;                                 // [CC][nk]  source spectrum
  float2 *fout = fin + (size_t)CC * nk;              // [NZ][LD]  Stolt output / FFT work
  const int tid = threadIdx.x;
  const int ncol = v.nx * v.ny;
  const int nclass = (v.nx / 2 + 1) * (v.ny / 2 + 1);
  const int q0 = blockIdx.x * CL;
  const int f = blockIdx.y;
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
    const int h2 = nk / 2;
    for (int e = tid; e < CC * h2; e += K3C_NT) {
      const int sl = e / h2, i = e - sl * h2;
      if (colof[sl] >= 0)
        reinterpret_cast<float4 *>(fin + sl * nk)[i] =
            __ldcs(reinterpret_cast<const float4 *>(wf + (size_t)colof[sl] * nk) + i);
    }
  } else {
    for (int e = tid; e < CC * nk; e += K3C_NT) {
      const int sl = e / nk, i = e - sl * nk;
      if (colof[sl] >= 0) fin[e] = __ldcs(wf + (size_t)colof[sl] * nk + i);
    }
  }
  __syncthreads();
  // 2. Stolt pull over the in-band (class, j) pairs, filter at the two taps
  //    folded into the weights (readings R2-R5, R9)
  const double rr = v.rref[f] * (1.0 / TWO_PI);
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
    sarfft2::fft<NZ, CC, LD, K3C_NT, +1, 0, true, (NZ == 512 ? 16 : 0)>(
        fout, v.tw_z, tid, load, [] {},
        [&](int c, int m, float2 x) {
          const int col = colof[c];
          if (col >= 0) __stcs(dst + (size_t)col * NZ + m, x);
        });
  } else {
    for (int i = tid; i < CC * NZ; i += K3C_NT) {
      const int sl = i / NZ, z = i - sl * NZ;
      if (colof[sl] >= 0) dst[(size_t)colof[sl] * NZ + z] = load(sl, z);
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
constexpr int K3P_G = 256;   // threads per consumer group
constexpr int K3P_NG = 2;    // consumer groups (alternate items)
constexpr int K3P_S = 3;     // ring stages
template <int NZ, int CL>
size_t k3pp_smem(int nk) {
  const size_t hdr = (sizeof(K3Hdr<CL>) + 15) & ~(size_t)15;
  return K3P_S * (hdr + (size_t)4 * CL * nk * sizeof(float2)) +
         K3P_NG * ((size_t)NZ * (4 * CL + 1)) * sizeof(float2) +
         ((size_t)NZ + nk) * sizeof(double) + (size_t)NZ * sizeof(float2);
}

template <int NZ, int CL, bool DO_IFFT, int BAR>
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
    const double rr = v.rref[f] * (1.0 / TWO_PI);
    // Stolt pull over the in-band (class, j) pairs only, the filter evaluated
    // at the two taps each pull uses and folded into the weights:
    //   O_j = (1-tau) H(k_i0) S_i0 + tau H(k_i0+1) S_i0+1
    int tot = 0;
#pragma unroll
    for (int cl = 0; cl < CL; ++cl) tot += h.jhi[cl] - h.jlo[cl] + 1;
    for (int idx = (v.dbg & 2) ? tot : gt; idx < tot; idx += K3P_G) {
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
    sarfft2::sync<BAR, K3P_G>();
    if (gt == 0) sartma::mbar_arrive(&empty[st]);  // stage (header + columns) consumed
    // inverse z-FFT (out-of-band rows read as zero), columns stored contiguously
    float2 *dst = v.w1 + (size_t)f * ncol * (size_t)NZ;
    auto load = [&](int c, int m) {
      return (m >= slo[c] && m <= shi[c]) ? fout[m * LD + c] : make_float2(0.f, 0.f);
    };
    if (DO_IFFT && !(v.dbg & 4)) {
      sarfft2::fft<NZ, CC, LD, K3P_G, +1, BAR, true, (NZ == 512 && CC == 8 ? 16 : 0)>(
          fout, tw, gt, load, [] {},
          [&](int c, int m, float2 x) {
            const int col = colofs[c];
            if (col >= 0) __stcs(dst + (size_t)col * NZ + m, x);
          });
    } else {
      for (int i = gt; i < CC * NZ; i += K3P_G) {
        const int sl = i / NZ, z = i - sl * NZ;
        if (sl < nu) dst[(size_t)colofs[sl] * NZ + z] = load(sl, z);
      }
    }
    sarfft2::sync<BAR, K3P_G>();  // fout / slot tables are rewritten by this group's next item
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
  float2 *tw = reinterpret_cast<float2 *>(kzs + NZ);              // [NZ]
  __shared__ __align__(8) uint64_t full[K3P_S], empty[K3P_S];
  __shared__ int colofs[K3P_NG][CC], slo[K3P_NG][CC], shi[K3P_NG][CC];
  const int tid = threadIdx.x;
  for (int i = tid; i < nk; i += NTH) ks[i] = v.k[i];
  for (int i = tid; i < NZ; i += NTH) {
    kzs[i] = v.kz[i];
    tw[i] = v.tw_z[i];
  }
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
    if (tid == K3P_NG * K3P_G) {  // producer
      const int hx = v.nx / 2 + 1, hy = v.ny / 2 + 1;
      const int nclass = hx * hy;
      unsigned n = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
        const int st = n % K3P_S;
        if (n >= K3P_S) sartma::mbar_wait(&empty[st], ((n / K3P_S) - 1) & 1);
        unsigned char *sb = ring + st * stage_bytes;
        K3Hdr<CL> &h = *reinterpret_cast<K3Hdr<CL> *>(sb);
        float2 *fin = reinterpret_cast<float2 *>(sb + hdr_bytes);
        const int f = item / nitems_f;
        const int q0 = (item - f * nitems_f) * CL;
        int cnt = 0;
        for (int cl = 0; cl < CL; ++cl) {
          const int q = q0 + cl;
          h.nmem[cl] = 0;
          h.kr2[cl] = 0.0;
          h.jlo[cl] = 0;
          h.jhi[cl] = -1;
          if (q >= nclass) continue;
          const SarClass &c = v.cls[q];
          h.kr2[cl] = c.kr2;
          h.jlo[cl] = c.jlo;
          h.jhi[cl] = c.jhi;
          for (int m = 0; m < c.nmem; ++m) {
            h.mslot[cl][h.nmem[cl]++] = cnt;
            h.clof[cnt] = cl;
            h.colof[cnt++] = c.col[m];
          }
        }
        h.nused = cnt;
        h.f = f;
        const float2 *wf = v.w0 + (size_t)f * ncol * (size_t)nk;
        sartma::mbar_arrive_expect_tx(&full[st], (uint32_t)cnt * (uint32_t)nk * 8u);
        for (int sl = 0; sl < cnt; ++sl)
          sartma::bulk_g2s(fin + sl * nk, wf + (size_t)h.colof[sl] * nk, (uint32_t)nk * 8u, &full[st]);
      }
    }
    return;
  }
  const int g = tid / K3P_G, gt = tid - g * K3P_G;
  float2 *fout = grp + g * grp_elems;
  if (g == 0)
    k3pp_consume<NZ, CL, DO_IFFT, 1>(v, nitems_f, 0, gt, ring, stage_bytes, hdr_bytes, fout, ks, kzs, tw, full, empty,
                                     colofs[0], slo[0], shi[0]);
  else
    k3pp_consume<NZ, CL, DO_IFFT, 2>(v, nitems_f, 1, gt, ring, stage_bytes, hdr_bytes, fout, ks, kzs, tw, full, empty,
                                     colofs[1], slo[1], shi[1]);
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
  const int nclass = (v.nx / 2 + 1) * (v.ny / 2 + 1);
  if (q >= nclass) return;
  const SarClass &c = v.cls[q];
  const int nm = c.nmem, nk = v.nk, ns = v.nz;
  const int ncol = v.nx * v.ny;
  const double kr2 = c.kr2;
  const double zoff = v.rref[f];   // z_s - Z_0 = (z_s - z_ref) + R_ref
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
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int item = tid + e * NT;
    if (ITEMS % NT != 0 && item >= ITEMS) continue;
    const int zz = item / NX, ix = item - zz * NX;
    const int z = zbase + zz;
    if (z >= nz) continue;
    int m = z + v.zroll;
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

// Persistent, TMA-pipelined K4b (n_z even, 32 <= nx <= 512).  Item = (frame,
// image row y, 16-wide z chunk): the [nx][16] tile of item i+1 is in flight
// (cp.async.bulk.tensor + mbarrier) while item i is inverse-transformed along
// x; the magnitudes (or scaled complex values) are transposed through a padded
// [16][nx+1] buffer with the x roll applied, so every image row segment is
// written with coalesced stores.
template <int NX, bool CPLX>
__global__ void __launch_bounds__(ntp_for(NX), ctas_for(NX))
    k4_xifft_mag_tma(const SarDeviceView v, const __grid_constant__ CUtensorMap tm, void *__restrict__ img,
                     int nzc, int nitems) {
  constexpr int NT = ntp_for(NX);
  constexpr int ROWS = NX < 256 ? NX : 256;
  constexpr int NBOX = NX / ROWS;
  constexpr uint32_t TILE_BYTES = NX * KC * sizeof(float2);
  using OT = typename std::conditional<CPLX, float2, float>::type;
  extern __shared__ __align__(128) float2 smk[];    // [2][NX][16] tiles, then [16][NX+1] output rows
  OT *ob = reinterpret_cast<OT *>(smk + 2 * (size_t)NX * KC);
  __shared__ __align__(8) uint64_t full[2];
  __shared__ float2 tw[NX];
  const int tid = threadIdx.x;
  const int nz = v.nz;
  for (int i = tid; i < NX; i += NT) tw[i] = v.tw_x[i];
  if (tid == 0) {
    sartma::mbar_init(&full[0], 1);
    sartma::mbar_init(&full[1], 1);
    sartma::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int item, int st) {
    const int zc = item % nzc, fy = item / nzc;  // fy = f*ny + y
    sartma::mbar_arrive_expect_tx(&full[st], TILE_BYTES);
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx)
      sartma::tma_load_3d(smk + (size_t)st * NX * KC + bx * ROWS * KC, &tm, zc * KC, bx * ROWS, fy, &full[st]);
  };
  const int rx = ((v.roll_x % NX) + NX) % NX;
  const int ry = ((v.roll_y % v.ny) + v.ny) % v.ny;
  const float sc = v.img_scale;
  int item = blockIdx.x;
  if (tid == 0 && item < nitems) issue(item, 0);
  for (int it = 0; item < nitems; ++it, item += gridDim.x) {
    const int st = it & 1;
    const int next = item + gridDim.x;
    if (tid == 0 && next < nitems) issue(next, st ^ 1);
    sartma::mbar_wait(&full[st], (it >> 1) & 1);
    float2 *tile = smk + (size_t)st * NX * KC;
    sarfft::tile_fft<NX, KC, KC, NT, +1>(tile, tw, tid);
    // transpose into output rows: ob[zz][ix] with ix = (a - r_x) mod nx
#pragma unroll
    for (int i = tid; i < NX * KC; i += NT) {
      const int a = i / KC, zz = i % KC;
      const float2 o = tile[i];
      const int ix = (a - rx) & (NX - 1);
      if constexpr (CPLX) {
        ob[zz * (NX + 1) + ix] = make_float2(o.x * sc, o.y * sc);
      } else {
        const float p = fmaf(o.x, o.x, o.y * o.y);
        ob[zz * (NX + 1) + ix] = p > 0.f ? p * rsqrtf(p) * sc : 0.f;   // |o| (rsqrt: 2 ulp)
      }
    }
    sartma::fence_proxy_async();
    __syncthreads();  // tile st is free (next-next load may overwrite it), ob complete
    const int zc = item % nzc, fy = item / nzc;
    const int f = fy / v.ny, y = fy - f * v.ny;
    int iy = y - ry;
    if (iy < 0) iy += v.ny;
    OT *outp = reinterpret_cast<OT *>(img) + ((size_t)f * nz * v.ny + iy) * NX;
    const size_t zstride = (size_t)v.ny * NX;
#pragma unroll
    for (int i = tid; i < NX * KC; i += NT) {
      const int zz = i / NX, ix = i % NX;
      const int z = zc * KC + zz;
      if (z < nz) {
        int m = z + v.zroll;
        if (m >= nz) m -= nz;
        outp[m * zstride + ix] = ob[zz * (NX + 1) + ix];
      }
    }
    __syncthreads();  // ob free
  }
}

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
constexpr int PB_NT = 256;    // consumer threads (+1 producer warp)
constexpr int PB_S = 2;       // ring stages
constexpr int PB_CL = 2;      // mirror classes per S item (<= 8 columns)
constexpr int PB_KC = 8;      // tile width of the Y / I items ([ny][8], 64-byte rows)

template <int NY, int NZ>
__host__ __device__ size_t passb_stage_bytes(int nk) {
  const size_t hdr = (sizeof(K3Hdr<PB_CL>) + 15) & ~(size_t)15;
  const size_t a = (size_t)NY * PB_KC * sizeof(float2), b = hdr + (size_t)4 * PB_CL * nk * sizeof(float2);
  return ((a > b ? a : b) + 127) & ~(size_t)127;
}
template <int NY, int NZ>
constexpr int passb_work() {
  return NY * PB_KC > NZ * (4 * PB_CL + 1) ? NY * PB_KC : NZ * (4 * PB_CL + 1);
}
template <int NY, int NZ>
size_t passb_smem(int nk) {
  return PB_S * passb_stage_bytes<NY, NZ>(nk) + (size_t)passb_work<NY, NZ>() * sizeof(float2) +
         (size_t)(NY + NZ) * sizeof(float2);
}

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void discard_l2(const void *p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

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

// --------------------------------------------------------- NUFFT mode ----
// SAR_GRID_NUFFT (reading R19, FGG-NUFFT of P:239-242).  K1n: one CTA per
// (16-wide k chunk, fine row jy of the 2ny x 2nx oversampled grid, frame).
// For each (pair, pose row) that can reach the fine row (host-built list) the
// CTA stages the pose row's samples rotated by e^{+j k beta} (Eq. (11)) and
// weighted by the row's Gaussian y-weight, plus each pose's x-weights; then
// every thread gathers into the fine-grid cells it owns (deterministic, no
// atomics).  Finally the fine row is transformed along x (N = 2nx), cropped
// to |a_s| < nx/2 and deconvolved by 1/Phi_x: Wh[f][jy][a][k].
// K2n: y-FFT over the 2ny fine rows, crop to |b_s| < ny/2, 1/Phi_y: W0.
constexpr int K1N_WT = 14;      // taps per axis: 2W + 2 with W = 6
constexpr int K1N_PCH = 256;    // poses staged at a time
constexpr int K1N_KC = 4;       // k values per CTA
constexpr int K1N_NT = 512;
template <int RX>
constexpr int k1n_br() { return RX >= 1024 ? 4 : 8; }   // fine rows per band (matches plan.cpp)

// One CTA = (k chunk of 4, band of BR fine rows, frame).  Thread (row r, k q,
// segment) owns the fine cells [seg*L, seg*L + L) x (r, q) in registers.  For
// each candidate (pair, pose row): stage the row's samples in fine-x order
// (host permutation) rotated by e^{+j k beta}, with each pose's x-weights and
// its y-weights for the band's rows; then every thread sweeps the sorted poses
// over its columns (positions may wrap by +-RX, reading R6).
template <int RX>
__global__ void __launch_bounds__(K1N_NT, 1) k1n_spread_xfft(const __grid_constant__ SarDeviceView v,
                                                             const float2 *__restrict__ s) {
  constexpr int BR = k1n_br<RX>();
  constexpr int CB = BR * K1N_KC;              // (row, k) pairs = FFT columns
  constexpr int SEGS = K1N_NT / CB;            // threads per (row, k)
  constexpr int L = RX / SEGS;                 // fine columns per thread
  extern __shared__ __align__(16) unsigned char smn[];
  const int npx = v.npx, nk = v.nk, W = v.nu_w;
  const int pch = npx < K1N_PCH ? npx : K1N_PCH;
  float2 *sval = reinterpret_cast<float2 *>(smn);                     // [pch][KC] staged samples
  float *wx = reinterpret_cast<float *>(sval + (size_t)pch * K1N_KC);  // [pch][WT]
  float *wyb = wx + (size_t)pch * K1N_WT;                             // [pch][BR]
  int *x0s = reinterpret_cast<int *>(wyb + (size_t)pch * BR);          // [pch] first tap column (no wrap)
  float2 *tile = reinterpret_cast<float2 *>(smn);                     // [RX][CB] (after the gather)
  __shared__ float2 twx[RX];
  const int tid = threadIdx.x;
  const int pair_idx = tid / SEGS, seg = tid - pair_idx * SEGS;
  const int r = pair_idx / K1N_KC, q = pair_idx - r * K1N_KC;
  const int c0 = seg * L;
  const int kc = blockIdx.x, band = blockIdx.y, f = blockIdx.z;
  const int RY = 2 * v.ny, NB = (RY + BR - 1) / BR;
  for (int i = tid; i < RX; i += K1N_NT) {
    float sn, cs;
    sincospif(-2.0f * (float)i / (float)RX, &sn, &cs);   // twiddles of the fine x-FFT
    twx[i] = make_float2(cs, sn);
  }
  const float inv2s2 = 0.5f / v.nu_s2;
  float2 acc[L];
#pragma unroll
  for (int m = 0; m < L; ++m) acc[m] = make_float2(0.f, 0.f);
  const int e0 = v.nu_off[f * NB + band], e1 = v.nu_off[f * NB + band + 1];
  for (int e = e0; e < e1; ++e) {
    const int code = __ldg(v.nu_cand + e);
    const int pr = code >> 16, iy = code & 0xffff;
    const int t = pr / v.nr, rr = pr - t * v.nr;
    const int jx2 = 2 * v.jx[pr];
    const size_t prow = (size_t)f * v.P + (size_t)iy * npx;
    const float2 *sg = s + (((size_t)(f * v.nt + t) * v.nr + rr) * v.P + (size_t)iy * npx) * nk;
    const float bp = v.no_comp ? 0.f : v.bpair[f * v.npair + pr];
    for (int p0 = 0; p0 < npx; p0 += K1N_PCH) {
      const int pn = npx - p0 < K1N_PCH ? npx - p0 : K1N_PCH;
      __syncthreads();   // the previous gather is done before the stage is rewritten
      for (int idx = tid; idx < pn * K1N_KC; idx += K1N_NT) {
        const int il = idx / K1N_KC, qq = idx - il * K1N_KC;
        const int ix = __ldg(v.nu_perm + prow + p0 + il);
        const int kq = kc * K1N_KC + qq;
        float2 val = make_float2(0.f, 0.f);
        if (kq < nk) {
          val = __ldcs(sg + (size_t)ix * nk + kq);
          if (!v.no_comp) {
            float turns = (__ldg(v.apose + prow + ix) + bp) * __ldg(v.kturn + kq);
            turns -= rintf(turns);
            float sn, cs;
            __sincosf(turns * 6.28318530717958647692f, &sn, &cs);
            val = cmul(val, make_float2(cs, sn));
          }
        }
        sval[idx] = val;
        if (qq == 0) {
          const float xf = (float)(2 * ix) + __ldg(v.nu_du + prow + ix);
          const int xb = (int)floorf(xf) - W;
          x0s[il] = xb + jx2;
#pragma unroll
          for (int tt = 0; tt < K1N_WT; ++tt) {
            const float dx = (float)(xb + tt) - xf;
            wx[il * K1N_WT + tt] = fabsf(dx) <= (float)W ? __expf(-dx * dx * inv2s2) : 0.f;
          }
          const float vf = (float)(2 * (iy + v.jy[pr])) + __ldg(v.nu_dv + prow + ix);
#pragma unroll
          for (int b = 0; b < BR; ++b) {
            float d = (float)(band * BR + b) - vf;
            d -= (float)RY * rintf(d / (float)RY);         // periodic fine rows (reading R6)
            wyb[il * BR + b] = fabsf(d) <= (float)W ? __expf(-d * d * inv2s2) : 0.f;
          }
        }
      }
      __syncthreads();
      // gather over the x-sorted poses: cell c gets tap c - x0 of the poses
      // with x0 <= c <= x0 + WT - 1, for the aliases c, c - RX, c + RX
      const int xlo = x0s[0], xhi = x0s[pn - 1] + K1N_WT - 1;
#pragma unroll
      for (int wrap = -1; wrap < 2; ++wrap) {
        const int cs = c0 + wrap * RX, ce = cs + L - 1;
        if (ce < xlo || cs > xhi) continue;
        // first pose whose footprint reaches cs (binary search, x0 ascending)
        int lo = 0, hi = pn;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (x0s[mid] + K1N_WT - 1 < cs) lo = mid + 1;
          else hi = mid;
        }
        for (int pp = lo; pp < pn; ++pp) {
          const int x0 = x0s[pp];
          if (x0 > ce) break;
          const float wyv = wyb[pp * BR + r];
          if (wyv == 0.f) continue;
          const float2 val = sval[pp * K1N_KC + q];
          const float2 vw = make_float2(val.x * wyv, val.y * wyv);
#pragma unroll
          for (int m = 0; m < L; ++m) {
            const int tt = cs + m - x0;
            if (tt >= 0 && tt < K1N_WT) {
              const float w = wx[pp * K1N_WT + tt];
              acc[m].x = fmaf(w, vw.x, acc[m].x);
              acc[m].y = fmaf(w, vw.y, acc[m].y);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  // the band's fine rows -> x-FFT (N = RX) over CB columns, crop, deconvolve
#pragma unroll
  for (int m = 0; m < L; ++m) tile[(c0 + m) * CB + pair_idx] = acc[m];
  __syncthreads();
  const int nx = v.nx;
  const int kmax = nk - kc * K1N_KC;
  sarfft2::fft<RX, CB, CB, K1N_NT, -1, 0, false>(
      tile, twx, tid, [&](int c, int n) { return tile[n * CB + c]; }, [] {},
      [&](int c, int n, float2 x) {
        const int as = n < RX / 2 ? n : n - RX;
        const int rb = c / K1N_KC, qb = c - rb * K1N_KC;
        const int jyf = band * BR + rb;
        if (qb < kmax && jyf < RY && as >= -nx / 2 && as < nx / 2) {
          const int a = as < 0 ? as + nx : as;
          const float d = __ldg(v.nu_decx + a);
          v.wh[((size_t)(f * RY + jyf) * nx + a) * (size_t)nk + kc * K1N_KC + qb] = make_float2(x.x * d, x.y * d);
        }
      });
}

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
  const float2 *src = v.wh + ((size_t)f * RY * nx + a) * (size_t)nk + kc * KC;
  const size_t row = (size_t)nx * nk;
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
          const float d = __ldg(v.nu_decy + b);
          dst[(size_t)b * row + c] = make_float2(x.x * d, x.y * d);
        }
      });
}

cudaError_t launch_nufft(const SarDeviceView &v, const float2 *data, cudaStream_t s) {
  const int nchunk = (v.nk + KC - 1) / KC;
  {
    const int pch = v.npx < K1N_PCH ? v.npx : K1N_PCH;
    switch (2 * v.nx) {
#define X(N)                                                                                        \
  case N: {                                                                                         \
    constexpr int BR = k1n_br<N>();                                                                 \
    const size_t stage = (size_t)pch * (K1N_KC * sizeof(float2) + (K1N_WT + BR) * sizeof(float) + sizeof(int)); \
    const size_t tile = (size_t)N * BR * K1N_KC * sizeof(float2);                                   \
    const size_t smem = stage > tile ? stage : tile;                                                \
    dim3 grid((v.nk + K1N_KC - 1) / K1N_KC, (2 * v.ny + BR - 1) / BR, v.F);                          \
    cudaError_t e = cudaFuncSetAttribute(k1n_spread_xfft<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                 \
    k1n_spread_xfft<N><<<grid, K1N_NT, smem, s>>>(v, data);                                          \
    e = cudaGetLastError();                                                                         \
    if (e != cudaSuccess) return e;                                                                 \
    break;                                                                                          \
  }
      X(64) X(128) X(256) X(512) X(1024)
#undef X
      default:
        return cudaErrorInvalidValue;
    }
  }
  dim3 grid(nchunk, v.nx, v.F);
  switch (2 * v.ny) {
#define X(N)                                                                                         \
  case N: {                                                                                          \
    const size_t smem = (size_t)N * KC * sizeof(float2);                                             \
    cudaError_t e = cudaFuncSetAttribute(k2n_yfft_crop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                  \
    k2n_yfft_crop<N><<<grid, sarfft2::nt_fft<N, KC>(), smem, s>>>(v);                                \
    return cudaGetLastError();                                                                       \
  }
    X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)
#undef X
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------ dispatch ----
#define SAR_SIZES(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)

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

cudaError_t launch_k1(const SarDeviceView &v, const float2 *data, bool fft, cudaStream_t s,
                      const CUtensorMap *tm_s, const CUtensorMap *tm_ap, int br, bool regacc, int num_sms) {
  if (fft && tm_s && tm_ap && v.nx >= 64 && v.nx <= 512 && v.k1_step_ok) {
    const int C = k1c_for(v.nx);
    const int nchunk = (v.nk + C - 1) / C;
    const int nitems = nchunk * v.ny * v.F;
    const int nbox = (v.npx + br - 1) / br;
    const int brmax = K1_BOX_BYTES / (C * 8);
    const size_t smem = (size_t)v.nx * C * sizeof(float2) + K1_STAGES * ((size_t)K1_BOX_BYTES + brmax * sizeof(float)) +
                        (size_t)v.nx * sizeof(float2);
    const int grid = nitems < num_sms ? nitems : num_sms;
    switch (v.nx) {
#define X(N)                                                                                          \
  case N: {                                                                                           \
    auto kern = regacc ? k1_correct_xfft_tma<N, true> : k1_correct_xfft_tma<N, false>;               \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                   \
    kern<<<grid, K1_NT + 32, smem, s>>>(v, *tm_s, *tm_ap, br, nbox, nitems);                               \
    return cudaGetLastError();                                                                        \
  }
      X(64) X(128) X(256) X(512)
#undef X
    }
  }
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
cudaError_t launch_mid(float2 *data, const float2 *tw, int F, int ny, int nx, int inner, cudaStream_t s,
                       const CUtensorMap *tm, int num_sms) {
  if (tm && ny <= 512 && !getenv("SAR_MID_OLD")) {
    const int nchunk = (inner + KC - 1) / KC;
    const int nitems = nchunk * nx * F;
    switch (ny) {
#define X(N)                                                                                       \
  case N: {                                                                                        \
    auto kern = k_fft_mid2<N, DIR>;                                                                \
    constexpr size_t smem = mid2_smem<N>();                                                        \
    if (smem > 40 * 1024) {                                                                        \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (e != cudaSuccess) return e;                                                              \
    }                                                                                              \
    const int maxg = num_sms * mid2_ctas<N>();                                                     \
    kern<<<nitems < maxg ? nitems : maxg, sarfft2::nt_fft<N, KC>() + 32, smem, s>>>(*tm, data, tw, nx, inner, \
                                                                                  nchunk, nitems); \
    return cudaGetLastError();                                                                     \
  }
      X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512)
#undef X
    }
    return cudaErrorInvalidValue;
  }
  if (tm && ny <= 512) {
    const int nchunk = (inner + KC - 1) / KC;
    const int nitems = nchunk * nx * F;
    const size_t smem = 2 * (size_t)ny * KC * sizeof(float2);
    switch (ny) {
#define X(N)                                                                                       \
  case N: {                                                                                        \
    auto kern = k_fft_mid_tma<N, DIR>;                                                             \
    if (smem > 40 * 1024) {                                                                        \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (e != cudaSuccess) return e;                                                              \
    }                                                                                              \
    const int maxg = num_sms * ctas_for(N);                                                        \
    kern<<<nitems < maxg ? nitems : maxg, ntp_for(N), smem, s>>>(*tm, tw, nx, nchunk, nitems);     \
    return cudaGetLastError();                                                                     \
  }
      SAR_SIZES(X)
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
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  kernel<<<grid, nt, smem, s>>>(v);
  return cudaGetLastError();
}

cudaError_t launch_k3(const SarDeviceView &v, bool ifft, cudaStream_t s, int num_sms) {
  if ((v.nk & 1) == 0 && v.nz >= 256 && !getenv("SAR_K3_PLAIN")) {
    const int nclass = (v.nx / 2 + 1) * (v.ny / 2 + 1);
    switch (v.nz) {
#define X(N)                                                                                                   \
  case N: {                                                                                                    \
    constexpr int CL = 2;                                                                                      \
    const size_t smem = k3pp_smem<N, CL>(v.nk);                                                                \
    if (smem > 225 * 1024) break;                                                                              \
    const int nitems_f = (nclass + CL - 1) / CL;                                                               \
    const int nitems = nitems_f * v.F;                                                                         \
    const int grid = nitems < num_sms ? nitems : num_sms;                                                      \
    auto kern = ifft ? k3_pp<N, CL, true> : k3_pp<N, CL, false>;                                               \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    if (e != cudaSuccess) return e;                                                                            \
    kern<<<grid, K3P_NG * K3P_G + 32, smem, s>>>(v, nitems_f);                                                 \
    return cudaGetLastError();                                                                                 \
  }
      X(256) X(512) X(1024)
#undef X
    }
  }
  const int nclass = (v.nx / 2 + 1) * (v.ny / 2 + 1);
  switch (v.nz) {
#define X(N)                                                                                                   \
  case N: {                                                                                                    \
    constexpr int CL = k3c_cl<N>();                                                                            \
    const size_t smem = k3c_smem<N>(v.nk);                                                                     \
    if (smem > 220 * 1024) return cudaErrorInvalidValue;                                                       \
    dim3 grid((nclass + CL - 1) / CL, v.F);                                                                    \
    auto kern = ifft ? k3_class<N, true> : k3_class<N, false>;                                                 \
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

cudaError_t launch_k4b(const SarDeviceView &v, void *img, bool cplx, cudaStream_t s, const CUtensorMap *tm,
                       int num_sms) {
  if (tm && v.nx <= 512 && !getenv("SAR_K4B_OLD")) {
    const int nzc = (v.nz + KC - 1) / KC;
    const int nitems = nzc * v.ny * v.F;
    switch (v.nx) {
#define X(N)                                                                                           \
  case N: {                                                                                            \
    auto kern = cplx ? k4_xifft_mag2<N, true> : k4_xifft_mag2<N, false>;                               \
    constexpr size_t smem = k4b2_smem<N, false>();                                                     \
    if (smem > 40 * 1024) {                                                                            \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (e != cudaSuccess) return e;                                                                  \
    }                                                                                                  \
    const int maxg = num_sms * k4b2_ctas<N>();                                                         \
    kern<<<nitems < maxg ? nitems : maxg, sarfft2::nt_fft<N, KC>() + 32, smem, s>>>(v, *tm, img, nzc, nitems); \
    return cudaGetLastError();                                                                         \
  }
      X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512)
#undef X
    }
  }
  if (tm && v.nx >= 32 && v.nx <= 512) {
    const int nzc = (v.nz + KC - 1) / KC;
    const int nitems = nzc * v.ny * v.F;
    const size_t smem = 2 * (size_t)v.nx * KC * sizeof(float2) + (size_t)KC * (v.nx + 1) * (cplx ? 8 : 4);
    switch (v.nx) {
#define X(N)                                                                                           \
  case N: {                                                                                            \
    auto kern = cplx ? k4_xifft_mag_tma<N, true> : k4_xifft_mag_tma<N, false>;                        \
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                    \
    const int cps = ctas_for(N) * smem <= 200 * 1024 ? ctas_for(N) : 1;                               \
    const int maxg = num_sms * cps;                                                                    \
    kern<<<nitems < maxg ? nitems : maxg, ntp_for(N), smem, s>>>(v, *tm, img, nzc, nitems);            \
    return cudaGetLastError();                                                                         \
  }
      X(32) X(64) X(128) X(256) X(512)
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
  const CUtensorMap *tm_s = nullptr;
  if (p->tma_ap) {
    if (p->tm_s_ptr != d_data) p->tma_s = sar_encode_input_map(p, d_data);
    if (p->tma_s) tm_s = &p->tm_s;
  }
  if (v.nufft) {
    // K1n (spread + fine x-FFT) and K2n (fine y-FFT + crop) replace K1 and K2;
    // their times are reported in the K1 and K2 slots
    SAR_CHECK(launch_nufft(v, data, s));
    if (ev) SAR_CHECK(cudaEventRecord(ev[1], s));
    if (ev) SAR_CHECK(cudaEventRecord(ev[2], s));
    if (stop_stage == 2) return SAR_OK;
    SAR_CHECK(launch_k3(v, stop_stage != 3, s, p->num_sms));
    if (ev) SAR_CHECK(cudaEventRecord(ev[3], s));
    if (stop_stage == 3) return SAR_OK;
    SAR_CHECK(launch_mid<+1>(v.w1, v.tw_y, v.F, v.ny, v.nx, v.nz, s, p->tma_mid1 ? &p->tm_w1_mid : nullptr,
                             p->num_sms));
    if (ev) SAR_CHECK(cudaEventRecord(ev[4], s));
    SAR_CHECK(launch_k4b(v, d_image, complex_out != 0, s, p->tma_rows1 ? &p->tm_w1_rows : nullptr, p->num_sms));
    if (ev) SAR_CHECK(cudaEventRecord(ev[5], s));
    return SAR_OK;
  }
  SAR_CHECK(launch_k1(v, data, stop_stage != 1, s, tm_s, p->tma_ap ? &p->tm_ap : nullptr, p->k1_br, p->k1_regacc,
                      p->num_sms));
  if (ev) SAR_CHECK(cudaEventRecord(ev[1], s));
  if (stop_stage == 1) return SAR_OK;
  if (p->fused) {
    // K2 + K3 + K4a as one kernel (its time is reported in the K3 slot)
    if (ev) SAR_CHECK(cudaEventRecord(ev[2], s));
    SAR_CHECK(launch_passb(v, &p->tm_w0_pb, &p->tm_w1_pb, p->d_items, p->n_items, p->d_cnt,
                           stop_stage == 2 || stop_stage == 3 ? stop_stage : 0,
                           stop_stage == 0 && p->passb_discard, s, p->num_sms));
    if (ev) SAR_CHECK(cudaEventRecord(ev[3], s));
    if (stop_stage == 2 || stop_stage == 3) return SAR_OK;
    if (ev) SAR_CHECK(cudaEventRecord(ev[4], s));
  } else {
    SAR_CHECK(launch_mid<-1>(v.w0, v.tw_y, v.F, v.ny, v.nx, v.nk, s, p->tma_mid0 ? &p->tm_w0_mid : nullptr,
                             p->num_sms));
    if (ev) SAR_CHECK(cudaEventRecord(ev[2], s));
    if (stop_stage == 2) return SAR_OK;
    if (v.mode2d) {
      const int nclass = (v.nx / 2 + 1) * (v.ny / 2 + 1);
      const int cpb = K3P2_NT / 32;
      k3_plane<<<dim3((nclass + cpb - 1) / cpb, v.F), K3P2_NT, 0, s>>>(v);
      SAR_CHECK(cudaGetLastError());
    } else {
      SAR_CHECK(launch_k3(v, stop_stage != 3, s, p->num_sms));
    }
    if (ev) SAR_CHECK(cudaEventRecord(ev[3], s));
    if (stop_stage == 3) return SAR_OK;
    SAR_CHECK(launch_mid<+1>(v.w1, v.tw_y, v.F, v.ny, v.nx, v.nz, s, p->tma_mid1 ? &p->tm_w1_mid : nullptr,
                             p->num_sms));
    if (ev) SAR_CHECK(cudaEventRecord(ev[4], s));
  }
  SAR_CHECK(launch_k4b(v, d_image, complex_out != 0, s, p->tma_rows1 ? &p->tm_w1_rows : nullptr, p->num_sms));
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

// ------------------------------------------------------- tensor maps ------
#include <cudaTypedefs.h>

namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 3-D map over a complex64 volume [d2][d1][d0] (d0 fastest), 8-byte elements.
bool encode3d(CUtensorMap *m, void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
              uint32_t b2) {
  auto enc = get_encode();
  if (!enc) return false;
  if ((d0 * 8) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 8, d0 * d1 * 8};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
}  // namespace

// 2-D map over a row-major [d1][d0] array of `esize`-byte elements
static bool encode2d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, uint64_t esize, uint64_t d0,
                     uint64_t d1, uint32_t b0, uint32_t b1) {
  auto enc = get_encode();
  if (!enc) return false;
  if ((d0 * esize) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {d0 * esize};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// raw samples viewed as [F*n_tx*n_rx*P rows][n_k] complex64, box [br rows][16]
bool sar_encode_input_map(sar_plan *p, const void *d_data) {
  const SarDeviceView &v = p->v;
  p->tm_s_ptr = d_data;
  const uint64_t rows = (uint64_t)v.F * v.nt * v.nr * v.P;
  return encode2d(&p->tm_s, d_data, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, v.nk, rows, k1c_for(v.nx), p->k1_br);
}

int sar_build_tensor_maps(sar_plan *p) {
  const SarDeviceView &v = p->v;
  p->tma_mid0 = p->tma_mid1 = p->tma_rows1 = false;
  if (v.F == 0 || getenv("SAR_NO_TMA")) return SAR_OK;
  const uint32_t rows = v.ny < 256 ? v.ny : 256;
  p->tma_mid0 = encode3d(&p->tm_w0_mid, v.w0, v.nk, v.nx, (uint64_t)v.F * v.ny, KC, 1, rows);
  p->tma_mid1 = encode3d(&p->tm_w1_mid, v.w1, v.nz, v.nx, (uint64_t)v.F * v.ny, KC, 1, rows);
  p->tma_pb = encode3d(&p->tm_w0_pb, v.w0, v.nk, v.nx, (uint64_t)v.F * v.ny, PB_KC, 1, rows) &&
              encode3d(&p->tm_w1_pb, v.w1, v.nz, v.nx, (uint64_t)v.F * v.ny, PB_KC, 1, rows);
  const uint32_t xr = v.nx < 256 ? v.nx : 256;
  p->tma_rows1 = encode3d(&p->tm_w1_rows, v.w1, v.nz, v.nx, (uint64_t)v.F * v.ny, KC, xr, 1);
  // K1: -2 d_z table [F*npy][npx] float32 with box [1][br]; input map per call
  const int brmax = K1_BOX_BYTES / (k1c_for(v.nx) * 8);
  p->k1_br = v.npx < brmax ? v.npx : brmax;
  p->k1_regacc = true;
  for (int i = 0; i < v.npair; ++i) p->k1_regacc = p->k1_regacc && v.jx[i] == 0;
  p->tma_ap = (v.npx % 4 == 0) && (v.nk % 2 == 0) && p->k1_br % 8 == 0 &&
              encode2d(&p->tm_ap, v.apose, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, v.npx, (uint64_t)v.F * v.npy,
                       p->k1_br, 1);
  p->tm_s_ptr = nullptr;
  p->tma_s = false;
  return SAR_OK;
}

// Fused pass B: decide, build the item list (see k_passb) and allocate it with
// the dependency counters.  Returns SAR_OK with p->fused = false when the
// geometry is not covered.
int sar_setup_passb(sar_plan *p) {
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
