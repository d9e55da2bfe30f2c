// membench.cu -- HBM read/copy bandwidth of the access patterns the path uses
// (row segments of C complex64 = 8C bytes at a fixed row stride), to choose
// tile shapes.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cstdio>
#include <cuda_runtime.h>

// CTA = (chunk of C columns, group of ROWS rows).  Each thread loads float2.
template <int C, int ROWS, int NT, bool COPY>
__global__ void seg(const float2 *__restrict__ in, float2 *__restrict__ out, long long row_stride, int ncol_chunks,
                    float *sink) {
  const int chunk = blockIdx.x % ncol_chunks;
  const long long grp = blockIdx.x / ncol_chunks;
  constexpr int ITEMS = C * ROWS;
  float2 acc = make_float2(0, 0);
#pragma unroll 4
  for (int it = threadIdx.x; it < ITEMS; it += NT) {
    const int c = it % C, r = it / C;
    const long long off = (grp * ROWS + r) * row_stride + (long long)chunk * C + c;
    float2 v = __ldcs(in + off);
    if (COPY) out[off] = v;
    else { acc.x += v.x; acc.y += v.y; }
  }
  if (!COPY && acc.x == 12345.f) *sink = acc.y;
}

__global__ void stream4(const float4 *__restrict__ in, float4 *__restrict__ out, long long n, float *sink, int copy) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float4 v = __ldcs(in + i);
    if (copy) out[i] = v;
    else { acc.x += v.x; }
  }
  if (acc.x == 12345.f) *sink = acc.y;
}

template <int C, int ROWS, int NT, bool COPY>
void run(const char *name, float2 *in, float2 *out, long long total, long long row_stride_elems, float *sink) {
  const int ncol_chunks = (int)(row_stride_elems / C);
  const long long nrows = total / row_stride_elems;
  const long long blocks = (long long)ncol_chunks * (nrows / ROWS);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) seg<C, ROWS, NT, COPY><<<(unsigned)blocks, NT>>>(in, out, row_stride_elems, ncol_chunks, sink);
  cudaEventRecord(a);
  const int reps = 5;
  for (int w = 0; w < reps; ++w) seg<C, ROWS, NT, COPY><<<(unsigned)blocks, NT>>>(in, out, row_stride_elems, ncol_chunks, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)total * 8 * (COPY ? 2 : 1) * reps;
  printf("%-40s C=%3d (%4d B) rows/CTA=%4d stride=%8lld B  %s  %7.1f GB/s\n", name, C, C * 8, ROWS,
         row_stride_elems * 8, COPY ? "copy" : "read", bytes / (ms * 1e-3) / 1e9);
}

int main() {
  const long long total = 1ll << 29;  // 512 Mi complex64 = 4 GiB
  float2 *in, *out;
  float *sink;
  cudaMalloc(&in, total * 8);
  cudaMalloc(&out, total * 8);
  cudaMalloc(&sink, 4);
  cudaMemset(in, 0, total * 8);
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int copy = 0; copy < 2; ++copy) {
      stream4<<<148 * 8, 512>>>((float4 *)in, (float4 *)out, total / 2, sink, copy);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) stream4<<<148 * 8, 512>>>((float4 *)in, (float4 *)out, total / 2, sink, copy);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("stream float4 %s: %.1f GB/s\n", copy ? "copy" : "read", total * 8.0 * (copy ? 2 : 1) * 5 / (ms * 1e-3) / 1e9);
    }
  }
  // K1-like: rows of 512 complex (4 KiB), segments of C
  run<16, 512, 512, false>("pose rows 4KiB", in, out, total, 512, sink);
  run<32, 512, 512, false>("pose rows 4KiB", in, out, total, 512, sink);
  run<64, 256, 512, false>("pose rows 4KiB", in, out, total, 512, sink);
  run<512, 8, 512, false>("pose rows 4KiB (full rows)", in, out, total, 512, sink);
  // K2-like: rows of 512*512 complex (2 MiB) stride
  run<16, 512, 512, true>("y rows 2MiB", in, out, total, 512 * 512, sink);
  run<32, 512, 512, true>("y rows 2MiB", in, out, total, 512 * 512, sink);
  run<64, 256, 512, true>("y rows 2MiB", in, out, total, 512 * 512, sink);
  run<16, 512, 512, true>("x rows 4KiB", in, out, total, 512, sink);
  run<32, 512, 512, true>("x rows 4KiB", in, out, total, 512, sink);
  run<64, 256, 512, true>("x rows 4KiB", in, out, total, 512, sink);
  run<512, 8, 512, true>("x full rows", in, out, total, 512, sink);
  // blocked layout: [chunk][row][16] contiguous 64 KiB tiles
  run<16, 512, 512, true>("contiguous 128B rows (stride 128B)", in, out, total, 16, sink);
  return 0;
}
