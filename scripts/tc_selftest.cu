// tc_selftest.cu -- checks the hand-built tcgen05 pieces the NUFFT spread uses
// (kind::tf32 MMA, SWIZZLE_NONE K-major shared-memory descriptors, TMEM
// alloc / ld / dealloc) against a CPU GEMM, single TF32 and 3xTF32.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tc_selftest scripts/tc_selftest.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int M = 128, N = 16, KC = 32;   // one K chunk of 32 (4 MMAs of K = 8)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// K-major, no swizzle: core matrix (8 rows x 16 B) at ((row/8) * (KC/4) + k/4) * 128 B
__device__ __forceinline__ int kmaj_off(int row, int k) { return ((row >> 3) * (KC / 4) + (k >> 2)) * 32 + (row & 7) * 4 + (k & 3); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;   // version (sm_100)
  return d;                 // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)            // D format F32
         | (2u << 7)          // A TF32
         | (2u << 10)         // B TF32
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);   // K-major A and B
}

template <int SPLIT>
__global__ void k_test(const float *A, const float *B, float *D) {
  __shared__ __align__(128) float sa[SPLIT][M * KC];
  __shared__ __align__(128) float sb[SPLIT][N * KC];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * KC; i += 128) {
    const int m = i / KC, k = i % KC;
    const float x = A[i], hi = tf32_rna(x);
    sa[0][kmaj_off(m, k)] = hi;
    if (SPLIT > 1) sa[1][kmaj_off(m, k)] = tf32_rna(x - hi);
  }
  for (int i = tid; i < N * KC; i += 128) {
    const int n = i / KC, k = i % KC;
    const float x = B[i], hi = tf32_rna(x);
    sb[0][kmaj_off(n, k)] = hi;
    if (SPLIT > 1) sb[1][kmaj_off(n, k)] = tf32_rna(x - hi);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_tf32(M, N);
    int first = 1;
    // 3xTF32: hi*hi + hi*lo + lo*hi
    for (int term = 0; term < (SPLIT > 1 ? 3 : 1); ++term) {
      const int ia = term == 2 ? 1 : 0, ib = term == 1 ? 1 : 0;
      for (int s = 0; s < KC / 8; ++s) {
        const uint64_t da = sdesc(smem_u32(&sa[ia][0]) + s * 256, 128, (KC / 4) * 128);
        const uint64_t db = sdesc(smem_u32(&sb[ib][0]) + s * 256, 128, (KC / 4) * 128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(first ? 0 : 1));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMAs
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < N; ++n) D[tid * N + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(M * KC), B(N * KC), D(M * N);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xffff) / 32768.f - 1.f; };
  for (auto &x : A) x = rnd();
  for (auto &x : B) x = rnd() * 0.5f + 0.5f;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  for (int split = 1; split <= 2; ++split) {
    CK(cudaMemset(dD, 0, D.size() * 4));
    if (split == 1) k_test<1><<<1, 128>>>(dA, dB, dD);
    else k_test<2><<<1, 128>>>(dA, dB, dD);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0, num = 0, den = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < KC; ++k) ref += (double)A[m * KC + k] * B[n * KC + k];
        const double d = D[m * N + n] - ref;
        maxerr = fmax(maxerr, fabs(d));
        maxref = fmax(maxref, fabs(ref));
        num += d * d;
        den += ref * ref;
      }
    printf("%s: rel L2 %.3e  max abs err %.3e (max |ref| %.3f)  D[0][0..3] %.5f %.5f %.5f %.5f\n",
           split == 1 ? "TF32  " : "3xTF32", sqrt(num / den), maxerr, maxref, D[0], D[1], D[2], D[3]);
  }
  return 0;
}
