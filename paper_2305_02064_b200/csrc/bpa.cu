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
// One thread per voxel, 128 voxels per CTA.  The CTA walks the poses in
// batches: the batch's sample rows [pair][pose][k] and element positions are
// staged in shared memory (every thread reads the same sample: broadcast
// loads), then for each (t, group of 4 receivers, pose) a thread forms the
// round-trip distance R in fp64, reduces the phases k_0 R and dk R to
// fractions of a turn in fp64 (|k R| reaches ~10^3 rad), and runs the k loop
// in paired fp32: acc += s_i * cur, cur *= step, re-seeding cur from the fp64
// phase every BPA_SEG samples so the recurrence error stays ~1e-6.  The four
// receivers are four independent chains (ILP); each k loop's fp32 sum is added
// to the voxel's fp64 total, so the rounding of the long sum does not grow
// with the number of terms.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "plan_internal.h"

namespace {

constexpr int BPA_NT = 128;   // voxels (threads) per CTA
constexpr int BPA_SEG = 32;   // k samples per phasor re-seed
constexpr int BPA_RG = 4;     // receivers per group (independent chains)

struct BpaArgs {
  const float2 *s;      // frame base: [npair][P][nk]
  const double *txw;    // [nt][P][3] Tx world positions minus the origin
  const double *rxw;    // [nr][P][3]
  const double *vox;    // [V][3] voxels minus the origin
  float2 *out;          // [V]
  long long V;
  int nt, nr, P, nk, PB;
  double kt0, dkt;      // k_0 / 2 pi, dk / 2 pi (turns per metre)
};

__device__ __forceinline__ float2 unit_phasor(double turns) {
  // exp(2 pi j turns): reduce in fp64, evaluate in fp32 (sincospif: <= 2 ulp)
  const float fr = (float)(turns - rint(turns));
  float2 r;
  sincospif(2.f * fr, &r.y, &r.x);
  return r;
}

__global__ void __launch_bounds__(BPA_NT) k_bpa(const BpaArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int npair = a.nt * a.nr;
  float2 *ss = reinterpret_cast<float2 *>(smraw);                                 // [npair][PB][nk]
  double *pt = reinterpret_cast<double *>(smraw + (size_t)npair * a.PB * a.nk * sizeof(float2));  // [nt][PB][3]
  double *prx = pt + (size_t)a.nt * a.PB * 3;                                      // [nr][PB][3]
  const int tid = threadIdx.x;
  long long v = (long long)blockIdx.x * BPA_NT + tid;
  const bool live = v < a.V;
  if (!live) v = a.V - 1;   // keeps the barriers uniform; its result is not stored
  const double vx = a.vox[v * 3], vy = a.vox[v * 3 + 1], vz = a.vox[v * 3 + 2];
  double tre = 0.0, tim = 0.0;

  for (int p0 = 0; p0 < a.P; p0 += a.PB) {
    const int cnt = min(a.PB, a.P - p0);
    __syncthreads();   // the previous batch is consumed
    const int per = cnt * a.nk;
    for (int e = tid; e < npair * per; e += BPA_NT) {
      const int pr = e / per, o = e - pr * per;
      ss[(size_t)pr * a.PB * a.nk + o] = __ldg(a.s + ((size_t)pr * a.P + p0) * a.nk + o);
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
      for (int r0 = 0; r0 < a.nr; r0 += BPA_RG) {
        double RR[BPA_RG];
#pragma unroll
        for (int j = 0; j < BPA_RG; ++j) {
          const int r = min(r0 + j, a.nr - 1);
          const double *q = prx + ((size_t)r * a.PB + pb) * 3;
          const double dx = vx - q[0], dy = vy - q[1], dz = vz - q[2];
          RR[j] = sqrt(dx * dx + dy * dy + dz * dz);
        }
        for (int t = 0; t < a.nt; ++t) {
          const double *q = pt + ((size_t)t * a.PB + pb) * 3;
          const double dx = vx - q[0], dy = vy - q[1], dz = vz - q[2];
          const double RT = sqrt(dx * dx + dy * dy + dz * dz);
          double ph0[BPA_RG], phd[BPA_RG];
          float2 step[BPA_RG], acc[BPA_RG];
          const float2 *row[BPA_RG];
#pragma unroll
          for (int j = 0; j < BPA_RG; ++j) {
            const double R = RT + RR[j];
            ph0[j] = a.kt0 * R;
            ph0[j] -= rint(ph0[j]);
            phd[j] = a.dkt * R;
            phd[j] -= rint(phd[j]);
            step[j] = unit_phasor(phd[j]);
            acc[j] = make_float2(0.f, 0.f);
            const int r = min(r0 + j, a.nr - 1);
            row[j] = ss + ((size_t)(t * a.nr + r) * a.PB + pb) * a.nk;
          }
          for (int i0 = 0; i0 < a.nk; i0 += BPA_SEG) {
            float2 cur[BPA_RG];
#pragma unroll
            for (int j = 0; j < BPA_RG; ++j) cur[j] = unit_phasor(ph0[j] + (double)i0 * phd[j]);
            const int i1 = min(i0 + BPA_SEG, a.nk);
            for (int i = i0; i < i1; ++i) {
#pragma unroll
              for (int j = 0; j < BPA_RG; ++j) {
                acc[j] = sark::cmac2(acc[j], row[j][i], cur[j]);
                cur[j] = sark::cmul2(cur[j], step[j]);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < BPA_RG; ++j)
            if (r0 + j < a.nr) {
              tre += (double)acc[j].x;
              tim += (double)acc[j].y;
            }
        }
      }
    }
  }
  if (live) a.out[v] = make_float2((float)tre, (float)tim);
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

  // poses per batch: ~16 KB of samples, one pose at least
  const size_t pose_bytes = (size_t)nt * nr * nk * sizeof(float2) + (size_t)(nt + nr) * 3 * sizeof(double);
  int PB = (int)(16384 / pose_bytes);
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

  DevBuf dt, dr, dv;
  if (cudaMalloc(&dt.p, txw.size() * 8) != cudaSuccess || cudaMalloc(&dr.p, rxw.size() * 8) != cudaSuccess ||
      cudaMalloc(&dv.p, vox.size() * 8) != cudaSuccess) {
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
  a.PB = PB;
  const double two_pi = 6.283185307179586476925286766559;
  a.kt0 = k0 / two_pi;
  a.dkt = dk / two_pi;
  if (smem > 40 * 1024 &&
      (e = cudaFuncSetAttribute(k_bpa, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return bcuda(e, "cudaFuncSetAttribute");
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms_out) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  const long long nblk = (n_voxels + BPA_NT - 1) / BPA_NT;
  k_bpa<<<(unsigned)nblk, BPA_NT, smem, s>>>(a);
  e = cudaGetLastError();
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
