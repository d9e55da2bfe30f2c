// tilebench.cu -- does the HBM layout of the intermediate volumes limit the
// mid-axis kernels (K2 / K4a / K4b)?  A K2-shaped persistent copy kernel
// (producer warp + TMA ring of [512][16] complex tiles, 512 consumer threads
// storing 128-byte rows) over a 1 GiB volume, with the tile read either as
// 512 rows of 128 B at a 2 MiB stride (today's [y][x][k] layout, 3-D TMA) or
// as one contiguous 64 KB block (a tiled [x][kc][y][16] layout, 1-D bulk
// copy), and the rows written at a 2 MiB, 4 KiB or 128 B (contiguous) stride.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tilebench scripts/tilebench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdint.h>

#include "../paper_2305_02064_b200/csrc/tma.cuh"

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

constexpr int N = 512, KC = 16, NCH = 32, NTC = 512;
constexpr uint32_t TILE = N * KC * 8;

template <int S, bool CIN, int OUT, bool IN4 = false>
__global__ void __launch_bounds__(NTC + 32, 1)
    tile_copy(const __grid_constant__ CUtensorMap tm, const float2 *__restrict__ in, float2 *__restrict__ out,
              int nitems, long long pitch) {
  extern __shared__ __align__(128) float2 ring[];
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      sartma::mbar_init(&full[i], 1);
      sartma::mbar_init(&empty[i], NTC / 32);
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
        const int chunk = item % NCH, x = item / NCH;
        sartma::mbar_arrive_expect_tx(&full[st], TILE);
        if (CIN) {
          sartma::bulk_g2s(ring + (size_t)st * N * KC, in + (size_t)item * N * KC, TILE, &full[st]);
        } else {
          for (int bx = 0; bx < 2; ++bx)
            if (IN4)
              sartma::tma_load_4d(ring + (size_t)st * N * KC + bx * 256 * KC, &tm, 0, chunk, x, bx * 256, &full[st]);
            else
            sartma::tma_load_3d(ring + (size_t)st * N * KC + bx * 256 * KC, &tm, chunk * KC, x, bx * 256,
                                &full[st]);
        }
      }
    }
    return;
  }
  unsigned n = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++n) {
    const int st = n % S;
    sartma::mbar_wait(&full[st], (n / S) & 1);
    const int chunk = item % NCH, x = item / NCH;
    const float4 *sv = reinterpret_cast<const float4 *>(ring + (size_t)st * N * KC);
    float4 r[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) r[it] = sv[it * NTC + tid];
    sartma::fence_proxy_async();
    __syncwarp();
    if ((tid & 31) == 0) sartma::mbar_arrive(&empty[st]);
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int e = it * NTC + tid, y = e >> 3, q = e & 7;
      size_t o;
      if (OUT == 0) o = (size_t)y * pitch + ((size_t)x * NCH + chunk) * KC;  // [y][x][k]: rows `pitch` apart
      else if (OUT == 1) o = (((size_t)x * NCH + chunk) * N + y) * KC;  // tiled: contiguous
      else o = (((size_t)x * N + y) * NCH + chunk) * KC;                 // [x][y][k]: rows 4 KiB apart
      reinterpret_cast<float4 *>(out + o)[q] = r[it];
    }
  }
}

template <int S, bool CIN, int OUT, bool IN4 = false>
int run(const char *name, const CUtensorMap &tm, float2 *in, float2 *out, long long pitch = (long long)N * N) {
  auto k = tile_copy<S, CIN, OUT, IN4>;
  const int smem = S * TILE;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int nitems = N * NCH;
  float best = 1e9f;
  for (int rep = 0; rep < 12; ++rep) {
    cudaEventRecord(a);
    k<<<148, NTC + 32, smem>>>(tm, in, out, nitems, pitch);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double bytes = 2.0 * (double)N * N * N * 8;
  printf("%-44s S=%d pitch+%lld B  %.4f ms  %.1f GB/s\n", name, S, (pitch - (long long)N * N) * 8, best, bytes / best / 1e6);
  return 0;
}

int main() {
  const size_t n = (size_t)N * N * N;
  float2 *in, *out;
  CK(cudaMalloc(&in, n * 8 + (size_t)N * 4200 * 8));
  CK(cudaMalloc(&out, n * 8 + (size_t)N * 4200 * 8));
  CK(cudaMemset(in, 0, n * 8));
  void *ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)N};   // k, x, y
  cuuint64_t strides[2] = {(cuuint64_t)N * 8, (cuuint64_t)N * N * 8};
  cuuint32_t box[3] = {KC, 1, 256};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, in, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const long long pads[5] = {0, 16, 32, 512, 4096 + 16};   // elements
  CUtensorMap tmp[5];
  for (int i = 0; i < 5; ++i) {
    cuuint64_t st2[2] = {(cuuint64_t)N * 8, (cuuint64_t)((long long)N * N + pads[i]) * 8};
    if (enc(&tmp[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, in, dims, st2, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int rep = 0; rep < 12; ++rep) {
    cudaEventRecord(a);
    cudaMemcpyAsync(out, in, n * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep >= 2 && ms < best) best = ms;
  }
  printf("%-44s      %.4f ms  %.1f GB/s\n", "cudaMemcpy D2D 1 GiB", best, 2.0 * n * 8 / best / 1e6);
  run<2, false, 0>("in 128B@2MiB (TMA) -> out 128B@2MiB", tm, in, out);
  run<2, true, 0>("in contiguous 64K  -> out 128B@2MiB", tm, in, out);
  run<2, false, 1>("in 128B@2MiB (TMA) -> out contiguous", tm, in, out);
  run<2, true, 1>("in contiguous 64K  -> out contiguous", tm, in, out);
  run<2, false, 2>("in 128B@2MiB (TMA) -> out 128B@4KiB", tm, in, out);
  run<2, true, 2>("in contiguous 64K  -> out 128B@4KiB", tm, in, out);
  run<3, false, 0>("in 128B@2MiB (TMA) -> out 128B@2MiB", tm, in, out);
  run<3, true, 0>("in contiguous 64K  -> out 128B@2MiB", tm, in, out);
  run<3, true, 1>("in contiguous 64K  -> out contiguous", tm, in, out);
  run<3, true, 2>("in contiguous 64K  -> out 128B@4KiB", tm, in, out);
  // K4b's input today ([y][x][z]: a tile's 512 rows 4 KiB apart) and in a
  // tiled K4a output [zc][x][y][16] (rows 64 KiB apart); 4-D maps
  // {16 zz, 32 zc, 512 y, 512 x}, box {16, 1, 1, 256}
  for (int i = 0; i < 2; ++i) {
    CUtensorMap t4;
    cuuint64_t d4[4] = {(cuuint64_t)KC, (cuuint64_t)NCH, (cuuint64_t)N, (cuuint64_t)N};
    cuuint64_t s4[3];
    if (i == 0) { s4[0] = KC * 8; s4[1] = (cuuint64_t)N * N * 8; s4[2] = (cuuint64_t)N * 8; }
    else { s4[0] = (cuuint64_t)N * N * KC * 8; s4[1] = KC * 8; s4[2] = (cuuint64_t)N * KC * 8; }
    cuuint32_t b4[4] = {KC, 1, 1, 256};
    cuuint32_t e4[4] = {1, 1, 1, 1};
    CUresult r = enc(&t4, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, in, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d (%d)\n", i, (int)r);
      continue;
    }
    run<2, false, 1, true>(i == 0 ? "K4b in today: 128B rows 4 KiB apart -> contig" : "K4b in tiled: 128B rows 64 KiB apart -> contig", t4, in, out);
    run<2, false, 2, true>(i == 0 ? "K4b in today: 128B rows 4 KiB apart -> 4KiB" : "K4b in tiled: 128B rows 64 KiB apart -> 4KiB", t4, in, out);
  }
  return 0;
}
