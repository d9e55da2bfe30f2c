// dsmem_bench.cu -- B200 measurements that decide the cluster design of the
// fused pass B: (1) how many 16/8/4/2-CTA clusters of
// one ~130-200 KB CTA per SM are co-resident; (2) distributed-shared-memory
// throughput per SM for thread loads (ld.shared::cluster.v4), thread stores
// (st.shared::cluster.v4) and TMA bulk pushes (cp.async.bulk
// shared::cluster.shared::cta) inside a 16-CTA cluster.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/dsmem_bench scripts/dsmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int BUF = 128 * 1024;

// every thread loads float4 from the shared memory of CTA (rank + 1 + it) % CS
template <int CS>
__global__ void k_ld(int iters, float *out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t base = smem_u32(sm);
  for (int i = threadIdx.x; i < BUF / 16; i += blockDim.x) reinterpret_cast<float4 *>(sm)[i] = make_float4(i, 1, 2, 3);
  cluster_sync();
  const uint32_t me = cluster_rank();
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const uint32_t peer = (me + 1 + (it % (CS - 1))) % CS;
    const uint32_t off = ((threadIdx.x + it * blockDim.x) * 16) % BUF;
    const uint32_t ra = mapa(base + off, peer);
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(ra));
    acc += v.x + v.w;
  }
  cluster_sync();
  if (acc == -1.f) out[0] = acc;
}

template <int CS>
__global__ void k_st(int iters, float *out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t base = smem_u32(sm);
  cluster_sync();
  const uint32_t me = cluster_rank();
  for (int it = 0; it < iters; ++it) {
    const uint32_t peer = (me + 1 + (it % (CS - 1))) % CS;
    const uint32_t off = ((threadIdx.x + it * blockDim.x) * 16) % BUF;
    const uint32_t ra = mapa(base + off, peer);
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(ra), "f"((float)it), "f"(1.f), "f"(2.f), "f"(3.f) : "memory");
  }
  cluster_sync();
  if (threadIdx.x == 0 && out == nullptr) out[0] = 0.f;
}

// local shared memory load throughput, same pattern (reference)
__global__ void k_local(int iters, float *out) {
  extern __shared__ __align__(16) unsigned char sm[];
  const uint32_t base = smem_u32(sm);
  for (int i = threadIdx.x; i < BUF / 16; i += blockDim.x) reinterpret_cast<float4 *>(sm)[i] = make_float4(i, 1, 2, 3);
  __syncthreads();
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const uint32_t off = ((threadIdx.x + it * blockDim.x) * 16) % BUF;
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(base + off));
    acc += v.x + v.w;
  }
  if (acc == -1.f) out[0] = acc;
}

// TMA bulk push: CTA r copies CH-byte chunks of its buffer A into buffer B of
// CTA (r+1) % CS, completion on the receiver's mbarrier; `rounds` rounds of
// BUF/2 bytes each, receiver-side barrier wait, then a cluster barrier so the
// sender may overwrite.
template <int CS, int CH>
__global__ void k_bulk(int rounds, float *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  unsigned char *A = sm, *B = sm + BUF / 2;
  const uint32_t me = cluster_rank();
  const uint32_t dst_rank = (me + 1) % CS;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync();
  const uint32_t rbar = mapa(smem_u32(&bar), dst_rank);
  const uint32_t rB = mapa(smem_u32(B), dst_rank);
  constexpr int NCH = (BUF / 2) / CH;
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(BUF / 2) : "memory");
    cluster_sync();  // every receiver armed before any push lands
    if (threadIdx.x < 32) {
      for (int c = threadIdx.x; c < NCH; c += 32)
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rB + c * CH),
            "r"(smem_u32(A + c * CH)), "r"(CH), "r"(rbar)
            : "memory");
    }
    // wait for my incoming data
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(r & 1) : "memory");
    }
  }
  cluster_sync();
  if (threadIdx.x == 0 && out == nullptr) out[0] = 0.f;
}

template <typename K>
int occ(K kern, int cs, size_t smem, int nt) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 64);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = -1;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
  if (e != cudaSuccess) printf("  occ err %s\n", cudaGetErrorString(e));
  return n;
}

template <typename K, typename... A>
float run(K kern, int cs, int nclusters, size_t smem, int nt, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * nclusters);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, kern, args...);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kern, args...);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    printf("  run error %s\n", cudaGetErrorString(e));
    return -1.f;
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d clock %d kHz\n", nsm, clk);
  float *out;
  CK(cudaMalloc(&out, 16));
  const size_t smem_big = 200 * 1024, smem_mid = 132 * 1024;
  auto setattr = [&](auto k) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_big);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  };
  setattr(k_ld<16>);
  setattr(k_ld<8>);
  setattr(k_ld<4>);
  setattr(k_ld<2>);
  setattr(k_st<16>);
  setattr(k_local);
  setattr(k_bulk<16, 256>);
  setattr(k_bulk<16, 4096>);
  setattr(k_bulk<16, 32768>);
  for (size_t sm : {smem_mid, smem_big}) {
    printf("smem %zu KB, 512 threads: max active clusters  cs16 %d  cs8 %d  cs4 %d  cs2 %d\n", sm / 1024,
           occ(k_ld<16>, 16, sm, 512), occ(k_ld<8>, 8, sm, 512), occ(k_ld<4>, 4, sm, 512), occ(k_ld<2>, 2, sm, 512));
  }
  const int nt = 512;
  const int iters = 4096;
  for (int cs : {16, 8, 4, 2}) {
    const int ncl = occ(cs == 16 ? k_ld<16> : cs == 8 ? k_ld<8> : cs == 4 ? k_ld<4> : k_ld<2>, cs, smem_mid, nt);
    float ms = -1;
    if (cs == 16) ms = run(k_ld<16>, 16, ncl, smem_mid, nt, iters, out);
    if (cs == 8) ms = run(k_ld<8>, 8, ncl, smem_mid, nt, iters, out);
    if (cs == 4) ms = run(k_ld<4>, 4, ncl, smem_mid, nt, iters, out);
    if (cs == 2) ms = run(k_ld<2>, 2, ncl, smem_mid, nt, iters, out);
    const double bytes_per_sm = (double)iters * nt * 16;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("ld.shared::cluster.v4  cs%-2d %d clusters: %.3f ms  %.1f B/clk/SM  aggregate %.1f TB/s\n", cs, ncl, ms,
           bytes_per_sm / cyc, bytes_per_sm * ncl * cs / (ms * 1e-3) / 1e12);
  }
  {
    const int ncl = occ(k_st<16>, 16, smem_mid, nt);
    float ms = run(k_st<16>, 16, ncl, smem_mid, nt, iters, out);
    const double bytes_per_sm = (double)iters * nt * 16;
    printf("st.shared::cluster.v4  cs16 %d clusters: %.3f ms  %.1f B/clk/SM\n", ncl, ms, bytes_per_sm / (ms * 1e-3 * clk * 1e3));
  }
  {
    float ms = run(k_local, 1, nsm, smem_mid, nt, iters, out);
    const double bytes_per_sm = (double)iters * nt * 16;
    printf("ld.shared.v4 local     %d CTAs: %.3f ms  %.1f B/clk/SM\n", nsm, ms, bytes_per_sm / (ms * 1e-3 * clk * 1e3));
  }
  for (int ch : {256, 4096, 32768}) {
    const int ncl = occ(k_bulk<16, 256>, 16, smem_mid, 128);
    const int rounds = 512;
    float ms = ch == 256 ? run(k_bulk<16, 256>, 16, ncl, smem_mid, 128, rounds, out)
                         : ch == 4096 ? run(k_bulk<16, 4096>, 16, ncl, smem_mid, 128, rounds, out)
                                      : run(k_bulk<16, 32768>, 16, ncl, smem_mid, 128, rounds, out);
    const double bytes_per_sm = (double)rounds * (BUF / 2);
    printf("cp.async.bulk push %5d B chunks cs16 %d clusters: %.3f ms  %.1f B/clk/SM (incl. a cluster barrier per 64 KB)\n", ch,
           ncl, ms, bytes_per_sm / (ms * 1e-3 * clk * 1e3));
  }
  return 0;
}
