// bpa.cu -- the GPU back-projection baseline (BPA): the
// paper's gold standard and comparison system, the
// matched filter of Eq. (9) with the exact round-trip distances of
// Eq. (2) and the ACTUAL (irregular) element positions:
//
//   o(v) = sum_{t,r,p,i} s[t,r,p,i] exp(+j k_i (|v - T_{t,p}| + |v - R_{r,p}|))
//
// O(V n_tx n_rx P n_k): ALU bound (one complex multiply-add per term plus the
// phasor that feeds it), not on the reconstruction hot path; it gives BPA
// timings and a physics check of the RMA image on configurations whose CPU
// brute force would take hours.
//
// One thread per 2 voxels (4 when n_k >= 384), 256 (512) voxels per CTA; gridDim.y splits the
// poses when there are few voxel CTAs (partial sums in fp64, reduced in a
// fixed order: deterministic).  The CTA walks its poses in batches: the
// batch's sample rows [pair][pose][k] (zero-padded to a multiple of 16) and
// element positions are staged in shared memory; every lane reads the same
// sample (broadcast loads), and a sample read once serves both voxels of the
// thread -- with one voxel per thread the kernel is bound by the shared-memory
// return path (a broadcast 8-byte load still fills 256 B of registers per
// warp), not by the FP32 pipe.  For each (t, r, pose, voxel) a thread forms
// the round-trip distance R in fp64, reduces the phases k_0 R and dk R to
// fractions of a turn in fp64 (|k R| reaches ~10^3 rad), builds the phasors
// w^e = exp(j e dk R), e = 1..8, in registers, and evaluates the k sum in
// blocks of 16 samples centred on e = 0:
//   sum_i s_i e^{j k_i R} = sum_a W_a sum_{e=-8..7} s_{16a+8+e} w^e,
//   W_a = e^{j (k_0 + (16a+8) dk) R},  w^{-e} = conj(w^e).
// With w^e = (c, d) and s = (x, y) the block sum needs no operand shuffles:
// A += (c,c)*(x,y) for every e, Bp += (d,d)*(x,y) for e > 0, Bn likewise for
// e < 0, and the sum is (A.x - (Bp-Bn).y, A.y + (Bp-Bn).x): two FFMA2 per
// term.  Per block one complex multiply-add and one step of W_a (W_a is
// re-seeded from the fp64 phase every BPA_RESEED blocks, so the recurrence
// error stays ~1e-6).  Each (t, r, pose) fp32 sum is added to the voxel's
// fp64 total, so the rounding of the long sum does not grow with the number
// of terms.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "plan_internal.h"

namespace {

constexpr int BPA_NT = 128;     // threads per CTA; BPA_NV voxels per thread (v, v + 128, ...): 2, or 4
                                // for long k rows (n_k >= 384: 216 registers, 8 warps per SM, half the
                                // shared-memory reads per term; measured Large 0.55 vs 0.47 of the FP32
                                // peak, Small 0.30 vs 0.35)
constexpr int BPA_NB = 16;      // k samples per block: e = -8 .. 7 around its centre
constexpr int BPA_H = BPA_NB / 2;
static_assert(BPA_H == 8, "the power tree below builds w^1 .. w^8");
constexpr int BPA_RESEED = 8;   // blocks per exact re-seed of the block phasor

struct BpaArgs {
  const float2 *s;      // frame base: [npair][P][nk]
  const double *txw;    // [nt][P][3] Tx world positions minus the origin
  const double *rxw;    // [nr][P][3]
  const double *vox;    // [V][3] voxels minus the origin
  float2 *out;          // [V] (nsplit == 1)
  double2 *part;        // [nsplit][V] partial sums (nsplit > 1)
  long long V;
  int nt, nr, P, nk, nkp, PB, nsplit;
  double kt0, dkt;      // k_0 / 2 pi, dk / 2 pi (turns per metre)
};

__device__ __forceinline__ float2 unit_phasor(double turns) {
  // exp(2 pi j turns): reduce in fp64, evaluate in fp32 (sincospif: <= 2 ulp)
  const float fr = (float)(turns - rint(turns));
  float2 r;
  sincospif(2.f * fr, &r.y, &r.x);
  return r;
}

template <int BPA_NV, int MINB>
__global__ void __launch_bounds__(BPA_NT, MINB) k_bpa(const BpaArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int npair = a.nt * a.nr;
  float2 *ss = reinterpret_cast<float2 *>(smraw);                                  // [npair][PB][nkp]
  double *pt = reinterpret_cast<double *>(smraw + (size_t)npair * a.PB * a.nkp * sizeof(float2));  // [nt][PB][3]
  double *prx = pt + (size_t)a.nt * a.PB * 3;                                       // [nr][PB][3]
  const int tid = threadIdx.x;
  long long v[BPA_NV];
  bool live[BPA_NV];
  double vx[BPA_NV], vy[BPA_NV], vz[BPA_NV], tre[BPA_NV], tim[BPA_NV];
#pragma unroll
  for (int j = 0; j < BPA_NV; ++j) {
    v[j] = ((long long)blockIdx.x * BPA_NV + j) * BPA_NT + tid;
    live[j] = v[j] < a.V;
    if (!live[j]) v[j] = a.V - 1;   // keeps the barriers uniform; its result is not stored
    vx[j] = a.vox[v[j] * 3], vy[j] = a.vox[v[j] * 3 + 1], vz[j] = a.vox[v[j] * 3 + 2];
    tre[j] = tim[j] = 0.0;
  }
  // this CTA's poses: split blockIdx.y of nsplit, in whole batches
  const int nbatch = (a.P + a.PB - 1) / a.PB;
  const int b_lo = (int)((long long)nbatch * blockIdx.y / a.nsplit);
  const int b_hi = (int)((long long)nbatch * (blockIdx.y + 1) / a.nsplit);

  for (int bt = b_lo; bt < b_hi; ++bt) {
    const int p0 = bt * a.PB;
    const int cnt = min(a.PB, a.P - p0);
    __syncthreads();   // the previous batch is consumed
    for (int e = tid; e < npair * cnt * a.nkp; e += BPA_NT) {
      const int i = e % a.nkp, rowi = e / a.nkp;        // rowi = pr * cnt + pb
      const int pr = rowi / cnt, pb = rowi - pr * cnt;
      float2 x = make_float2(0.f, 0.f);
      if (i < a.nk) x = __ldg(a.s + ((size_t)pr * a.P + p0 + pb) * a.nk + i);
      ss[((size_t)pr * a.PB + pb) * a.nkp + i] = x;
    }
    for (int e = tid; e < a.nt * cnt * 3; e += BPA_NT) {
      const int t = e / (cnt * 3), o = e - t * cnt * 3;
      pt[(size_t)t * a.PB * 3 + o] = a.txw[((size_t)t * a.P + p0) * 3 + o];
    }
    for (int e = tid; e < a.nr * cnt * 3; e += BPA_NT) {
      const int r = e / (cnt * 3), o = e - r * cnt * 3;
      prx[(size_t)r * a.PB * 3 + o] = a.rxw[((size_t)r * a.P + p0) * 3 + o];
    }
    __syncthreads();

    for (int pb = 0; pb < cnt; ++pb) {
      for (int r = 0; r < a.nr; ++r) {
        const double *qr = prx + ((size_t)r * a.PB + pb) * 3;
        double RR[BPA_NV];
#pragma unroll
        for (int j = 0; j < BPA_NV; ++j) {
          const double dx = vx[j] - qr[0], dy = vy[j] - qr[1], dz = vz[j] - qr[2];
          RR[j] = sqrt(dx * dx + dy * dy + dz * dz);
        }
        for (int t = 0; t < a.nt; ++t) {
          const double *q = pt + ((size_t)t * a.PB + pb) * 3;
          // per voxel: cc[e-1] = (c,c), dd[e-1] = (d,d) of w^e = (c,d), e = 1..8
          float2 cc[BPA_NV][BPA_H], dd[BPA_NV][BPA_H], Wstep[BPA_NV], Wa[BPA_NV], acc[BPA_NV];
          double ph0[BPA_NV], phd[BPA_NV];
#pragma unroll
          for (int j = 0; j < BPA_NV; ++j) {
            const double tx = vx[j] - q[0], ty = vy[j] - q[1], tz = vz[j] - q[2];
            const double R = RR[j] + sqrt(tx * tx + ty * ty + tz * tz);
            ph0[j] = a.kt0 * R;
            ph0[j] -= rint(ph0[j]);
            phd[j] = a.dkt * R;
            phd[j] -= rint(phd[j]);
            // powers w^1 .. w^8 by a product tree of depth 3 (w^2, w^4 by
            // squaring), not a chain of 7: shorter dependency and less rounding
            float2 wp[BPA_H];
            wp[0] = unit_phasor(phd[j]);
            wp[1] = sark::cmul2(wp[0], wp[0]);
            wp[2] = sark::cmul2(wp[1], wp[0]);
            wp[3] = sark::cmul2(wp[1], wp[1]);
            wp[4] = sark::cmul2(wp[3], wp[0]);
            wp[5] = sark::cmul2(wp[3], wp[1]);
            wp[6] = sark::cmul2(wp[3], wp[2]);
            wp[7] = sark::cmul2(wp[3], wp[3]);
#pragma unroll
            for (int e = 0; e < BPA_H; ++e) {
              cc[j][e] = make_float2(wp[e].x, wp[e].x);
              dd[j][e] = make_float2(wp[e].y, wp[e].y);
            }
            Wstep[j] = unit_phasor((double)BPA_NB * phd[j]);   // w^16, from the fp64 phase
            acc[j] = make_float2(0.f, 0.f);
            Wa[j] = make_float2(1.f, 0.f);
          }
          const float2 *row = ss + ((size_t)(t * a.nr + r) * a.PB + pb) * a.nkp;
          for (int blk = 0; blk * BPA_NB < a.nk; ++blk) {
            if (blk % BPA_RESEED == 0) {
#pragma unroll
              for (int j = 0; j < BPA_NV; ++j)
                Wa[j] = unit_phasor(ph0[j] + (double)(blk * BPA_NB + BPA_H) * phd[j]);
            }
            const float2 *rb = row + blk * BPA_NB + BPA_H;   // e = 0
            float2 A0[BPA_NV], A1[BPA_NV], Bp[BPA_NV], Bn[BPA_NV];
            const float2 s0 = rb[0], sm8 = rb[-BPA_H];
#pragma unroll
            for (int j = 0; j < BPA_NV; ++j) {
              A0[j] = s0;                                              // e = 0: w^0 = 1
              A1[j] = __fmul2_rn(cc[j][BPA_H - 1], sm8);               // e = -8
              Bn[j] = __fmul2_rn(dd[j][BPA_H - 1], sm8);
              Bp[j] = make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int e = 1; e < BPA_H; ++e) {
              const float2 sp = rb[e], sn = rb[-e];
#pragma unroll
              for (int j = 0; j < BPA_NV; ++j) {
                A0[j] = __ffma2_rn(cc[j][e - 1], sp, A0[j]);
                A1[j] = __ffma2_rn(cc[j][e - 1], sn, A1[j]);
                Bp[j] = __ffma2_rn(dd[j][e - 1], sp, Bp[j]);
                Bn[j] = __ffma2_rn(dd[j][e - 1], sn, Bn[j]);
              }
            }
#pragma unroll
            for (int j = 0; j < BPA_NV; ++j) {
              const float2 A = __fadd2_rn(A0[j], A1[j]);
              const float bx = Bp[j].x - Bn[j].x, by = Bp[j].y - Bn[j].y;
              acc[j] = sark::cmac2(acc[j], make_float2(A.x - by, A.y + bx), Wa[j]);
              Wa[j] = sark::cmul2(Wa[j], Wstep[j]);
            }
          }
#pragma unroll
          for (int j = 0; j < BPA_NV; ++j) {
            tre[j] += (double)acc[j].x;
            tim[j] += (double)acc[j].y;
          }
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < BPA_NV; ++j)
    if (live[j]) {
      if (a.nsplit == 1) a.out[v[j]] = make_float2((float)tre[j], (float)tim[j]);
      else a.part[(size_t)blockIdx.y * a.V + v[j]] = make_double2(tre[j], tim[j]);
    }
}

// sum of the pose splits in split order
__global__ void k_bpa_reduce(const double2 *__restrict__ part, float2 *__restrict__ out, long long V, int nsplit) {
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  double re = 0.0, im = 0.0;
  for (int sidx = 0; sidx < nsplit; ++sidx) {
    const double2 x = part[(size_t)sidx * V + v];
    re += x.x;
    im += x.y;
  }
  out[v] = make_float2((float)re, (float)im);
}

int bfail(int status, const std::string &msg) {
  sar_set_error(msg);
  return status;
}
int bcuda(cudaError_t e, const char *what) {
  sar_set_error(std::string("CUDA: ") + cudaGetErrorString(e) + " (" + what + ")");
  return SAR_ERR_CUDA;
}

struct DevBuf {
  void *p = nullptr;
  ~DevBuf() { cudaFree(p); }
};

}  // namespace

extern "C" int sar_bpa(const sar_geom_desc *g, int32_t frame, const void *d_data, const double *h_voxels,
                       int64_t n_voxels, void *d_out, sar_stream stream, float *ms_out) {
  if (!g) return bfail(SAR_ERR_INVALID_ARG, "geometry descriptor is NULL");
  if (g->n_tx < 1 || g->n_rx < 1 || g->n_tx * g->n_rx > SAR_MAX_PAIRS)
    return bfail(SAR_ERR_INVALID_ARG, "n_tx, n_rx >= 1 and n_tx*n_rx <= SAR_MAX_PAIRS");
  if (g->npx < 1 || g->npy < 1) return bfail(SAR_ERR_INVALID_ARG, "npx, npy must be >= 1");
  if (g->n_k < 2 || g->n_k > SAR_MAX_NK) return bfail(SAR_ERR_INVALID_ARG, "n_k out of range");
  if (frame < 0 || frame >= g->n_frames) return bfail(SAR_ERR_INVALID_ARG, "frame out of range");
  if (!g->tx_xyz || !g->rx_xyz || !g->scan_xyz || !g->k) return bfail(SAR_ERR_INVALID_ARG, "NULL geometry array");
  if (n_voxels < 0) return bfail(SAR_ERR_INVALID_ARG, "n_voxels < 0");
  if (ms_out) *ms_out = 0.f;
  if (n_voxels == 0) return SAR_OK;
  if (!d_data || !h_voxels || !d_out) return bfail(SAR_ERR_INVALID_ARG, "NULL buffer");
  const int nt = g->n_tx, nr = g->n_rx, nk = g->n_k;
  const long long P = (long long)g->npx * g->npy;
  if (P * nt * nr * (long long)g->n_frames >= (1LL << 31))
    return bfail(SAR_ERR_UNSUPPORTED, "n_frames * n_tx * n_rx * poses >= 2^31 sample rows");
  // uniform, ascending k (as sar_plan_create; the k loop steps by dk)
  const double k0 = g->k[0], dk = (g->k[nk - 1] - g->k[0]) / (nk - 1);
  if (!(k0 > 0.0) || !(dk > 0.0)) return bfail(SAR_ERR_GEOMETRY, "k must be positive and ascending");
  for (int i = 0; i < nk; ++i)
    if (fabs(g->k[i] - (k0 + i * dk)) > 1e-9 * g->k[nk - 1]) return bfail(SAR_ERR_GEOMETRY, "k is not uniform");

  // poses per batch: ~24 KB of staged samples (rows padded to whole blocks), one
  // pose at least
  const int nkp = (nk + BPA_NB - 1) / BPA_NB * BPA_NB;
  const size_t pose_bytes = (size_t)nt * nr * nkp * sizeof(float2) + (size_t)(nt + nr) * 3 * sizeof(double);
  int PB = (int)(24576 / pose_bytes);
  if (PB < 1) PB = 1;
  if (PB > P) PB = (int)P;
  const size_t smem = PB * pose_bytes;
  if (smem > 200 * 1024) return bfail(SAR_ERR_UNSUPPORTED, "one pose's sample rows exceed 200 KB of shared memory");

  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != g->device) {
    cudaError_t e = cudaSetDevice(g->device);
    if (e != cudaSuccess) return bcuda(e, "cudaSetDevice");
  }
  struct Restore {
    int prev, dev;
    ~Restore() {
      if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
  } restore{prev, g->device};
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, g->device);
  if (e != cudaSuccess) return bcuda(e, "cudaGetDeviceProperties");
  if (prop.major != 10) return bfail(SAR_ERR_UNSUPPORTED, "device is not sm_100 (B200)");

  // positions relative to the frame's mean pose (fp64 on the host), so the
  // device differences are formed from small numbers
  const double *scan = g->scan_xyz + (size_t)frame * P * 3;
  double c[3] = {0, 0, 0};
  for (long long p = 0; p < P; ++p)
    for (int d = 0; d < 3; ++d) c[d] += scan[p * 3 + d];
  for (int d = 0; d < 3; ++d) c[d] /= (double)P;
  std::vector<double> txw((size_t)nt * P * 3), rxw((size_t)nr * P * 3), vox((size_t)n_voxels * 3);
  for (int t = 0; t < nt; ++t)
    for (long long p = 0; p < P; ++p)
      for (int d = 0; d < 3; ++d) txw[((size_t)t * P + p) * 3 + d] = (scan[p * 3 + d] - c[d]) + g->tx_xyz[t * 3 + d];
  for (int r = 0; r < nr; ++r)
    for (long long p = 0; p < P; ++p)
      for (int d = 0; d < 3; ++d) rxw[((size_t)r * P + p) * 3 + d] = (scan[p * 3 + d] - c[d]) + g->rx_xyz[r * 3 + d];
  for (long long v = 0; v < n_voxels; ++v)
    for (int d = 0; d < 3; ++d) vox[(size_t)v * 3 + d] = h_voxels[v * 3 + d] - c[d];

  // few voxel CTAs: split the pose batches over gridDim.y (~6 CTAs per SM wanted)
  const int NV = nk >= 384 ? 4 : 2;
  const long long nblk = (n_voxels + BPA_NT * NV - 1) / (BPA_NT * NV);
  const long long nbatch = (P + PB - 1) / PB;
  long long nsplit = (6LL * prop.multiProcessorCount + nblk - 1) / nblk;
  if (nsplit > nbatch) nsplit = nbatch;
  if (nsplit > 65535) nsplit = 65535;
  if (nsplit < 1) nsplit = 1;
  DevBuf dt, dr, dv, dp;
  if (cudaMalloc(&dt.p, txw.size() * 8) != cudaSuccess || cudaMalloc(&dr.p, rxw.size() * 8) != cudaSuccess ||
      cudaMalloc(&dv.p, vox.size() * 8) != cudaSuccess ||
      (nsplit > 1 && cudaMalloc(&dp.p, (size_t)nsplit * n_voxels * sizeof(double2)) != cudaSuccess)) {
    cudaGetLastError();
    return bfail(SAR_ERR_OOM, "device allocation of the BPA tables failed");
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((e = cudaMemcpyAsync(dt.p, txw.data(), txw.size() * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(dr.p, rxw.data(), rxw.size() * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(dv.p, vox.data(), vox.size() * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return bcuda(e, "table upload");

  BpaArgs a;
  a.s = static_cast<const float2 *>(d_data) + (size_t)frame * nt * nr * P * nk;
  a.txw = static_cast<const double *>(dt.p);
  a.rxw = static_cast<const double *>(dr.p);
  a.vox = static_cast<const double *>(dv.p);
  a.out = static_cast<float2 *>(d_out);
  a.V = n_voxels;
  a.nt = nt;
  a.nr = nr;
  a.P = (int)P;
  a.nk = nk;
  a.nkp = nkp;
  a.PB = PB;
  a.nsplit = (int)nsplit;
  a.part = static_cast<double2 *>(dp.p);
  const double two_pi = 6.283185307179586476925286766559;
  a.kt0 = k0 / two_pi;
  a.dkt = dk / two_pi;
  void (*kern)(const BpaArgs) = NV == 4 ? k_bpa<4, 2> : k_bpa<2, 3>;
  if (smem > 40 * 1024 &&
      (e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return bcuda(e, "cudaFuncSetAttribute");
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms_out) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  kern<<<dim3((unsigned)nblk, (unsigned)nsplit), BPA_NT, smem, s>>>(a);
  e = cudaGetLastError();
  if (e == cudaSuccess && nsplit > 1) {
    k_bpa_reduce<<<(unsigned)((n_voxels + 255) / 256), 256, 0, s>>>(a.part, a.out, n_voxels, (int)nsplit);
    e = cudaGetLastError();
  }
  if (ms_out) cudaEventRecord(e1, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (ms_out) {
    if (e == cudaSuccess) cudaEventElapsedTime(ms_out, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (e != cudaSuccess) return bcuda(e, "k_bpa");
  return SAR_OK;
}
