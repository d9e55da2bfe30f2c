// k1bench.cu -- how fast can K1's raw-sample stream go?  The memory side of
// K1 alone: a persistent CTA per SM (or two), a producer warp issuing K1's
// TMA boxes ([br poses][16 k] of the [pairs * P][n_k] raw tensor, item =
// (pose row vy, 16-wide k chunk), jobs = (pair, box)) into an S-stage
// mbarrier ring, consumer warps that read each stage once (a running sum, so
// the reads are real) and hand it back; optionally each item ends with a
// 64 KB store of its [512][16] tile to a W0-shaped volume.  Large geometry:
// 12 pairs, 512 x 512 poses, n_k = 512 (12 GiB).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/k1bench scripts/k1bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2305_02064_b200/csrc/tma.cuh"

constexpr int NK = 512, NX = 512, NY = 512, NPAIR = 12, KC = 16, NCH = NK / KC;
constexpr long long P = (long long)NX * NY;

template <int S, int BR, int NCW, int STORE>
__global__ void __launch_bounds__(NCW * 32 + 32, 1)
    k1_stream(const __grid_constant__ CUtensorMap tm, float2 *__restrict__ w0, float *sink, int nitems) {
  constexpr uint32_t BOX = BR * KC * 8;
  constexpr int NB = NX / BR;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      sartma::mbar_init(&full[i], 1);
      sartma::mbar_init(&empty[i], NCW);
    }
    sartma::fence_barrier_init();
  }
  __syncthreads();
  if (tid >= NCW * 32) {
    if (tid == NCW * 32) {
      unsigned n = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int kc = item % NCH, vy = item / NCH;
        for (int pr = 0; pr < NPAIR; ++pr)
          for (int b = 0; b < NB; ++b, ++n) {
            const int st = n % S;
            if (n >= S) sartma::mbar_wait(&empty[st], ((n / S) - 1) & 1);
            sartma::mbar_arrive_expect_tx(&full[st], BOX);
            sartma::tma_load_2d(sm + (size_t)st * BOX, &tm, kc * KC, (int)(pr * P + (long long)vy * NX + b * BR),
                                &full[st]);
          }
      }
    }
    return;
  }
  float acc = 0.f;
  unsigned n = 0;
  const int lane = tid & 31;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    for (int j = 0; j < NPAIR * NB; ++j, ++n) {
      const int st = n % S;
      sartma::mbar_wait(&full[st], (n / S) & 1);
      const float4 *sv = reinterpret_cast<const float4 *>(sm + (size_t)st * BOX);
      for (int i = tid; i < (int)(BOX / 16); i += NCW * 32) {
        const float4 q = sv[i];
        acc += q.x + q.y + q.z + q.w;
      }
      sartma::fence_proxy_async();
      __syncwarp();
      if (lane == 0) sartma::mbar_arrive(&empty[st]);
    }
    if (STORE == 1) {   // today's W0 [vy][x][k]: 512 rows of 128 B, 4 KiB apart
      const int kc = item % NCH, vy = item / NCH;
      float2 *out = w0 + (size_t)vy * NX * NK + kc * KC;
      for (int i = tid; i < NX * KC; i += NCW * 32) out[(size_t)(i >> 4) * NK + (i & 15)] = make_float2(acc, 0.f);
    } else if (STORE == 2) {   // tiled W0 [vy][kc][x][16]: the item's 64 KB contiguous
      float2 *out = w0 + (size_t)item * NX * KC;
      for (int i = tid; i < NX * KC; i += NCW * 32) out[i] = make_float2(acc, 0.f);
    } else if (STORE == 3) {   // tiled, one 64 KB bulk store from shared memory
      float2 *tile = reinterpret_cast<float2 *>(sm + (size_t)S * BOX);
      if (tid == 0) sartma::bulk_wait_read0();
      asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
      for (int i = tid; i < NX * KC; i += NCW * 32) tile[i] = make_float2(acc, 0.f);
      sartma::fence_proxy_async();
      asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
      if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(w0 + (size_t)item * NX * KC),
                     "r"(sartma::smem_u32(tile)), "r"(NX * KC * 8)
                     : "memory");
        sartma::bulk_commit();
      }
    }
  }
  if (STORE == 3 && tid == 0) sartma::bulk_wait0();
  if (acc == 12345.f) sink[0] = acc;
}

template <int S, int BR, int NCW, int STORE>
void run(const CUtensorMap *tms, float2 *w0, float *sink, int ctas_per_sm) {
  auto k = k1_stream<S, BR, NCW, STORE>;
  const int smem = S * BR * KC * 8 + (STORE == 3 ? NX * KC * 8 : 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nitems = NY * NCH;
  const CUtensorMap &tm = tms[BR == 256 ? 0 : BR == 128 ? 1 : 2];
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(a);
    k<<<148 * ctas_per_sm, NCW * 32 + 32, smem>>>(tm, w0, sink, nitems);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep >= 1 && ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  const double rd = (double)NPAIR * P * NK * 8, wr = STORE ? (double)NY * NX * NK * 8 : 0.0;
  printf("S=%d box=[%3d][16] %2.0f KB  in flight %3d KB/CTA  %d CTA/SM  %2d consumer warps  %s  %.4f ms  read %.1f GB/s  total %.1f GB/s %s\n",
         S, BR, BR * KC * 8 / 1024.0, S * BR * KC * 8 / 1024, ctas_per_sm, NCW, STORE == 0 ? "no store    " : STORE == 1 ? "W0 rows@4KiB" : STORE == 2 ? "W0 tiled    " : "W0 tiled TMA", best,
         rd / best / 1e6, (rd + wr) / best / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const size_t rows = (size_t)NPAIR * P;
  float2 *raw, *w0;
  float *sink;
  if (cudaMalloc(&raw, rows * NK * 8) != cudaSuccess || cudaMalloc(&w0, (size_t)NY * NX * NK * 8) != cudaSuccess ||
      cudaMalloc(&sink, 64) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(raw, 0, rows * NK * 8);
  void *ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  CUtensorMap tms[3];
  const int brs[3] = {256, 128, 64};
  for (int i = 0; i < 3; ++i) {
    cuuint64_t dims[2] = {(cuuint64_t)NK, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)NK * 8};
    cuuint32_t box[2] = {KC, (cuuint32_t)brs[i]};
    cuuint32_t es[2] = {1, 1};
    if (enc(&tms[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, raw, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
  }
  for (int rep = 0; rep < 2; ++rep) {
    run<4, 256, 16, 0>(tms, w0, sink, 1);
    run<4, 256, 16, 1>(tms, w0, sink, 1);
    run<4, 256, 16, 2>(tms, w0, sink, 1);
    run<4, 256, 16, 3>(tms, w0, sink, 1);
    run<3, 256, 16, 1>(tms, w0, sink, 1);
    run<5, 256, 16, 1>(tms, w0, sink, 1);
    run<8, 128, 16, 1>(tms, w0, sink, 1);
    run<8, 128, 16, 3>(tms, w0, sink, 1);
  }
  return 0;
}
