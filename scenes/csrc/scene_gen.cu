// scene_gen.cu -- CUDA synthesis of the frequency-domain echo of Eq. (9)
// with Eq. (2) distances, for workloads too
// large to synthesise on the CPU (Freehand, Large, Realtime).
//
// INPUT GENERATOR ONLY: this library is not part of the reconstruction path
// and holds none of the method's arithmetic.  It re-implements the NumPy
// generator of scenes/__init__.py (synthesize_cpu) and the counter-based
// noise of scenes/rng.py; tests compare the two on small scenes.
//
//   s[f,t,r,p,i] = sum_n amp_n exp(-j k_i (|tx_w - q_n| + |rx_w - q_n|)) + noise
//
// fp64 distances; the phase of the first k of each 32-wide chunk is reduced in
// fp64 and the remaining 31 come from an fp32 phasor recurrence.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr int GK = 32;    // k per thread
constexpr int GNT = 128;  // threads per CTA
constexpr int GTILE = 256;  // scatterers staged per smem tile

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double uniform53(uint64_t b) {
  return ((double)(b >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

// grid: x = rows-of-this-frame / GNT, y = k chunks, z = frame
__global__ void __launch_bounds__(GNT)
    k_echo(float2 *__restrict__ out, int nt, int nr, int P, int nk, const double *__restrict__ tx,
           const double *__restrict__ rx, const double *__restrict__ scan, const double *__restrict__ scat,
           int nsc, double k0, double dk, unsigned long long key, double sigma) {
  __shared__ double sq[GTILE][5];
  const int f = blockIdx.z;
  const int rows = nt * nr * P;
  const int row = blockIdx.x * GNT + threadIdx.x;
  const bool active = row < rows;
  const int kb = blockIdx.y * GK;
  int t = 0, r = 0, p = 0;
  double txw[3] = {0, 0, 0}, rxw[3] = {0, 0, 0};
  if (active) {
    p = row % P;
    const int tr = row / P;
    t = tr / nr;
    r = tr % nr;
    const double *ps = scan + ((size_t)f * P + p) * 3;
    for (int d = 0; d < 3; ++d) {
      txw[d] = ps[d] + tx[3 * t + d];
      rxw[d] = ps[d] + rx[3 * r + d];
    }
  }
  float2 acc[GK];
#pragma unroll
  for (int i = 0; i < GK; ++i) acc[i] = make_float2(0.f, 0.f);
  const double *sf = scat + (size_t)f * nsc * 5;
  const double kstart = k0 + (double)kb * dk;
  for (int n0 = 0; n0 < nsc; n0 += GTILE) {
    const int cnt = min(GTILE, nsc - n0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < cnt * 5; idx += GNT) sq[idx / 5][idx % 5] = sf[(size_t)n0 * 5 + idx];
    __syncthreads();
    if (!active) continue;
    for (int n = 0; n < cnt; ++n) {
      const double ax = txw[0] - sq[n][0], ay = txw[1] - sq[n][1], az = txw[2] - sq[n][2];
      const double bx = rxw[0] - sq[n][0], by = rxw[1] - sq[n][1], bz = rxw[2] - sq[n][2];
      const double R = sqrt(ax * ax + ay * ay + az * az) + sqrt(bx * bx + by * by + bz * bz);
      double t0 = -kstart * R * (1.0 / 6.283185307179586476925286766559);
      t0 -= rint(t0);
      double t1 = -dk * R * (1.0 / 6.283185307179586476925286766559);
      t1 -= rint(t1);
      float s0, c0, s1, c1;
      sincospif((float)(2.0 * t0), &s0, &c0);
      sincospif((float)(2.0 * t1), &s1, &c1);
      const float ar = (float)sq[n][3], ai = (float)sq[n][4];
      float2 cur = make_float2(ar * c0 - ai * s0, ar * s0 + ai * c0);
#pragma unroll
      for (int i = 0; i < GK; ++i) {
        acc[i].x += cur.x;
        acc[i].y += cur.y;
        const float nx = cur.x * c1 - cur.y * s1;
        cur.y = cur.x * s1 + cur.y * c1;
        cur.x = nx;
      }
    }
  }
  if (!active) return;
  const size_t base = (((size_t)f * nt + t) * nr + r) * P + p;
  for (int i = 0; i < GK; ++i) {
    const int k = kb + i;
    if (k >= nk) break;
    const size_t idx = base * nk + k;
    float2 v = acc[i];
    if (sigma > 0) {
      const uint64_t c0 = (uint64_t)key + 2ull * (uint64_t)idx;
      const double u1 = uniform53(splitmix64(c0)), u2 = uniform53(splitmix64(c0 + 1));
      const double rr = sqrt(-2.0 * log(u1)) * (sigma / sqrt(2.0));
      double sn, cs;
      sincospi(2.0 * u2, &sn, &cs);
      v.x = (float)((double)v.x + rr * cs);
      v.y = (float)((double)v.y + rr * sn);
    }
    out[idx] = v;
  }
}

}  // namespace

extern "C" int scene_echo(void *d_out, int F, int nt, int nr, int P, int nk, const double *d_tx,
                          const double *d_rx, const double *d_scan, const double *d_scat, int nsc, double k0,
                          double dk, unsigned long long key, double sigma, void *stream) {
  if (F == 0) return 0;
  dim3 grid((nt * nr * P + GNT - 1) / GNT, (nk + GK - 1) / GK, F);
  k_echo<<<grid, GNT, 0, (cudaStream_t)stream>>>((float2 *)d_out, nt, nr, P, nk, d_tx, d_rx, d_scan, d_scat,
                                                  nsc, k0, dk, key, sigma);
  return (int)cudaGetLastError();
}
