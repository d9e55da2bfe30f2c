// pipeline.cu -- enqueues the kernels of the reconstruction path (one
// translation unit per kernel family) and builds the TMA tensor maps.  Citation keys: P:n = PAPER.md line n; readings R1..R17 are in
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
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost a pointer test unless a tool is attached
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "common.cuh"

using namespace sark;

namespace sark {
int resident_ctas(const void *kern, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void *, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(kern, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    n = 1;
  }
  n = n < 1 ? 1 : n;
  cache[key] = n;
  return n;
}
}  // namespace sark

// Enqueue the path for frames [f0, f0 + nf) (one frame wave; the workspace
// holds its frames from 0).  d_image points at frame f0 of the image.
// stop_stage: 0 = full; 1 = K1 without the x-FFT; 2 = K1+K2; 3 = K1+K2+K3
// without the z-IFFT.  ev (optional, 6 events) brackets the kernels.
int sar_launch_pipeline(sar_plan *p, const void *d_data, void *d_image, cudaStream_t s, int stop_stage,
                        int complex_out, cudaEvent_t *ev, int f0, int nf) {
  SarDeviceView vw = p->v;
  vw.f0 = f0;
  vw.F = nf;
  const SarDeviceView &v = vw;
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
  // NVTX: one range per kernel launch of the path (ncu --nvtx / any NVTX tool
  // can filter on them); popped on every exit of its scope
  struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
  };
  NvtxRange whole("sar_reconstruct: path");
  if (ev) SAR_CHECK(cudaEventRecord(ev[0], s));
  const CUtensorMap *tm_s = nullptr;
  if (p->tma_ap) {
    if (p->tm_s_ptr != d_data) p->tma_s = sar_encode_input_map(p, d_data);
    if (p->tma_s) tm_s = &p->tm_s;
  }
  if (v.nufft) {
    // the spread (K1s) and the fine x/y FFTs + crop (x-FFT, K2n) replace K1
    // and K2; their times are reported in the K1 and K2 slots
    const CUtensorMap *tmf = p->tma_fine ? &p->tm_fine : nullptr;
    {
      NvtxRange r("K1s NUFFT spread");
      SAR_CHECK(launch_nufft(v, data, s, tmf, p->num_sms, 1));
    }
    if (ev) SAR_CHECK(cudaEventRecord(ev[1], s));
    NvtxRange r("fine x-FFT + K2n");
    SAR_CHECK(launch_nufft(v, data, s, tmf, p->num_sms, 2));
  } else {
    {
      NvtxRange r("K1 correct + x-FFT");
      SAR_CHECK(launch_k1(v, data, stop_stage != 1, s, tm_s, p->tma_ap ? &p->tm_ap : nullptr, p->k1_br,
                          p->k1_regacc, p->num_sms));
    }
    if (ev) SAR_CHECK(cudaEventRecord(ev[1], s));
    if (stop_stage == 1) return SAR_OK;
    // debug stage 2 dumps the whole spectrum; otherwise rows of skipped
    // columns are not stored
    // (K2 keeps per-element stores: TMA stores of its live row boxes measured
    // slower, 0.366 vs 0.341 ms on Large; K4a below gains from them)
    NvtxRange r("K2 y-FFT");
    SAR_CHECK(launch_mid<-1>(v.w0, v.tw_y, v.F, v.ny, v.nx, v.nk, s, p->tma_mid0 ? &p->tm_w0_mid : nullptr,
                             p->num_sms, nullptr, stop_stage == 2 ? nullptr : v.liveb));
  }
  if (ev) SAR_CHECK(cudaEventRecord(ev[2], s));
  if (stop_stage == 2) return SAR_OK;
  // skipped columns are not written by K3: zero them for the stage-3 dump
  if (stop_stage == 3 && v.liveb)
    SAR_CHECK(cudaMemsetAsync(v.w1, 0, (size_t)v.F * v.ny * v.nx * v.nz * sizeof(float2), s));
  {
    NvtxRange r("K3 filter + Stolt + z-IFFT");
    if (v.mode2d) {
      SAR_CHECK(launch_k3_plane(v, s));
    } else {
      SAR_CHECK(launch_k3(v, stop_stage != 3, s, p->num_sms));
    }
  }
  if (ev) SAR_CHECK(cudaEventRecord(ev[3], s));
  if (stop_stage == 3) return SAR_OK;
  {
    NvtxRange r("K4a y-IFFT");
    SAR_CHECK(launch_mid<+1>(v.w1, v.tw_y, v.F, v.ny, v.nx, v.nz, s, p->tma_mid1 ? &p->tm_w1_mid : nullptr,
                             p->num_sms, nullptr, v.liveb, p->tma_mid1 && K4A_ROWS == 32 ? &p->tm_w1_mid : nullptr));
  }
  if (ev) SAR_CHECK(cudaEventRecord(ev[4], s));
  NvtxRange r4("K4b x-IFFT + magnitude");
  SAR_CHECK(launch_k4b(v, d_image, complex_out != 0, s, p->tma_rows1 ? &p->tm_w1_rows : nullptr, p->num_sms));
  if (ev) SAR_CHECK(cudaEventRecord(ev[5], s));
  return SAR_OK;
}

int sar_launch_stolt_index(sar_plan *p, const int32_t *d_cols, int n, int32_t *d_i0, float *d_tau,
                           cudaStream_t s) {
  cudaError_t e = launch_stolt_index(p->v, d_cols, n, d_i0, d_tau, s);
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
// 4-D map over a complex64 array [d3][d2][d1][d0] (d0 fastest)
bool encode4d(CUtensorMap *m, const void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b0,
              uint32_t b1, uint32_t b2, uint32_t b3) {
  auto enc = get_encode();
  if (!enc) return false;
  if ((d0 * 8) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  cuuint64_t dims[4] = {d0, d1, d2, d3};
  cuuint64_t strides[3] = {d0 * 8, d0 * d1 * 8, d0 * d1 * d2 * 8};
  cuuint32_t box[4] = {b0, b1, b2, b3};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
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

// ------------------------------------------------------- CUDA graphs ----
// SAR_CUDA_GRAPH.  The library links the static CUDA runtime while PyTorch
// loads its own shared one, and the runtime's stream capture failed in that
// arrangement (round 1); the capture and the graph calls here go straight to
// the driver (entry points looked up once), on a non-blocking stream of the
// plan, so the legacy default stream of the caller is never captured.
namespace {
struct GraphApi {
  CUresult (*begin)(CUstream, CUstreamCaptureMode) = nullptr;
  CUresult (*end)(CUstream, CUgraph *) = nullptr;
  CUresult (*inst)(CUgraphExec *, CUgraph, unsigned long long) = nullptr;
  CUresult (*launch)(CUgraphExec, CUstream) = nullptr;
  CUresult (*gdestroy)(CUgraph) = nullptr;
  CUresult (*edestroy)(CUgraphExec) = nullptr;
  bool ok = false;
};
const GraphApi &graph_api() {
  static GraphApi g;
  static bool tried = false;
  if (!tried) {
    tried = true;
    auto get = [](const char *name, void **fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    g.ok = get("cuStreamBeginCapture", (void **)&g.begin) && get("cuStreamEndCapture", (void **)&g.end) &&
           get("cuGraphInstantiateWithFlags", (void **)&g.inst) && get("cuGraphLaunch", (void **)&g.launch) &&
           get("cuGraphDestroy", (void **)&g.gdestroy) && get("cuGraphExecDestroy", (void **)&g.edestroy);
  }
  return g;
}
}  // namespace

void sar_graph_destroy(sar_plan *p) {
  if (p->graph_exec) {
    const GraphApi &g = graph_api();
    if (g.ok) g.edestroy(static_cast<CUgraphExec>(p->graph_exec));
    p->graph_exec = nullptr;
  }
}

int sar_graph_reconstruct(sar_plan *p, const void *d_data, void *d_image, cudaStream_t s) {
  const GraphApi &g = graph_api();
  if (!g.ok) {
    sar_set_error("CUDA graph driver entry points unavailable");
    return SAR_ERR_UNSUPPORTED;
  }
  if (!p->graph_exec || p->g_data != d_data || p->g_image != d_image) {
    sar_graph_destroy(p);
    // the capture stream must not overlap work the caller's stream still
    // has in flight on the plan's workspace
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      sar_set_error(std::string("CUDA: ") + cudaGetErrorString(e));
      return SAR_ERR_CUDA;
    }
    CUstream cs = reinterpret_cast<CUstream>(p->cap_stream);
    if (g.begin(cs, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL) != CUDA_SUCCESS) {
      sar_set_error("cuStreamBeginCapture failed");
      return SAR_ERR_CUDA;
    }
    const int st = sar_enqueue_call(p, d_data, d_image, p->cap_stream);
    CUgraph graph = nullptr;
    const CUresult ce = g.end(cs, &graph);
    if (st != SAR_OK) {
      if (graph) g.gdestroy(graph);
      return st;
    }
    if (ce != CUDA_SUCCESS || !graph) {
      sar_set_error("cuStreamEndCapture failed");
      return SAR_ERR_CUDA;
    }
    CUgraphExec exec = nullptr;
    const CUresult ie = g.inst(&exec, graph, 0);
    g.gdestroy(graph);
    if (ie != CUDA_SUCCESS) {
      sar_set_error("cuGraphInstantiate failed");
      return SAR_ERR_CUDA;
    }
    p->graph_exec = exec;
    p->g_data = d_data;
    p->g_image = d_image;
  }
  if (g.launch(static_cast<CUgraphExec>(p->graph_exec), reinterpret_cast<CUstream>(s)) != CUDA_SUCCESS) {
    sar_set_error("cuGraphLaunch failed");
    return SAR_ERR_CUDA;
  }
  return SAR_OK;
}

// raw samples viewed as [F*n_tx*n_rx*P rows][n_k] complex64, box [br rows][16]
bool sar_encode_input_map(sar_plan *p, const void *d_data) {
  const SarDeviceView &v = p->v;
  p->tm_s_ptr = d_data;
  const uint64_t rows = (uint64_t)v.F * v.nt * v.nr * v.P;
  return encode2d(&p->tm_s, d_data, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, v.nk, rows, k1c_for(v.nx), p->k1_br);
}

// Slab plans (workspace = the slabs only) skip the whole-image workspace maps
// and build K1's.
int sar_build_tensor_maps(sar_plan *p) {
  const SarDeviceView &v = p->v;
  p->tma_mid0 = p->tma_mid1 = p->tma_rows1 = p->tma_fine = p->tma_ap = false;
  if (v.F == 0 || v.force_plain) return SAR_OK;
  if (p->slab_world == 0) {
    const uint32_t rows = v.ny < 256 ? v.ny : 256, rows1 = v.ny < K4A_ROWS ? v.ny : K4A_ROWS;   // K2 / K4a boxes
    const uint64_t wf = (uint64_t)p->wave;   // the workspace holds one frame wave
    p->tma_mid0 = encode3d(&p->tm_w0_mid, v.w0, v.nk, v.nx, wf * v.ny, KC, 1, rows);
    p->tma_mid1 = encode3d(&p->tm_w1_mid, v.w1, v.nz, v.nx, wf * v.ny, KC, 1, rows1);
    if (v.nufft) {
      // fine grid [F*2ny][2nx][nk]: x-FFT boxes {16 k, 1, <=256 fine columns}
      const uint32_t rx = 2 * v.nx, fr = rx < 256 ? rx : 256;
      p->tma_fine = encode3d(&p->tm_fine, v.wh, v.nk, 1, (uint64_t)v.F * 2 * v.ny * rx, KC, 1, fr);
    }
    const uint32_t xr = v.nx < 256 ? v.nx : 256;
    p->tma_rows1 = encode3d(&p->tm_w1_rows, v.w1, v.nz, v.nx, wf * v.ny, KC, xr, 1);
  }
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


// ------------------------------------------------ slab decomposition ----
namespace {
// Destination of every block: d[h] (this rank's pack buffer + h*dhs, or --
// exchange by peer stores -- block h's slot in rank h's receive buffer,
// mapped into this process over NVLink).
struct BlockDst {
  char *d[SAR_MAX_SLAB];
};

// d[h] + r*dp  <-  src + h*shs + r*sp, Wb bytes per (h, r), for h < G, r < H:
// the packs / unpack of the slab exchanges (16-byte vectors, streaming)
__global__ void k_block_copy(const BlockDst dst, const char *__restrict__ src, unsigned G, unsigned H, unsigned V,
                             long long shs, long long sp, long long dp) {
  const unsigned total = G * H * V;   // < 2^31 (checked by the launcher)
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned q = i / V, v = i - q * V;
    const unsigned h = q / H, r = q - h * H;
    const float4 x = __ldcs(reinterpret_cast<const float4 *>(src + h * shs + r * sp) + v);
    __stcs(reinterpret_cast<float4 *>(dst.d[h] + r * dp) + v, x);
  }
}

cudaError_t block_copy(const BlockDst &dst, const void *src, int G, long long H, long long Wb, long long shs,
                       long long sp, long long dp, int num_sms, cudaStream_t s) {
  bool vec = !(Wb % 16 || shs % 16 || sp % 16 || dp % 16 || (double)G * H * (Wb / 16) >= 2147483648.0);
  for (int h = 0; h < G; ++h) vec = vec && (reinterpret_cast<uintptr_t>(dst.d[h]) % 16 == 0);
  if (!vec) {
    for (int h = 0; h < G; ++h) {
      cudaError_t e = cudaMemcpy2DAsync(dst.d[h], dp, static_cast<const char *>(src) + h * shs, sp, Wb, H,
                                        cudaMemcpyDefault, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const int V = (int)(Wb / 16);
  const long long total = (long long)G * H * V;
  const long long want = (total + 255) / 256;
  const int grid = (int)(want < 8LL * num_sms ? want : 8LL * num_sms);
  k_block_copy<<<grid > 0 ? grid : 1, 256, 0, s>>>(dst, static_cast<const char *>(src), (unsigned)G, (unsigned)H,
                                                  (unsigned)V, shs, sp, dp);
  return cudaGetLastError();
}

// blocks of a contiguous [G][...] buffer (block stride hs bytes)
BlockDst dst_packed(void *base, int G, long long hs) {
  BlockDst d{};
  for (int h = 0; h < G; ++h) d.d[h] = static_cast<char *>(base) + h * hs;
  return d;
}
// this rank's block slot in every peer's receive buffer
BlockDst dst_peers(void *const *peers, int G, int rank, long long hs) {
  BlockDst d{};
  for (int h = 0; h < G; ++h) d.d[h] = static_cast<char *>(peers[h]) + rank * hs;
  return d;
}
}  // namespace

// Buffers of a slab plan (the whole-image workspace is reused): W0 holds the
// K1 output of this rank's lattice rows [ny'][nx][nk] and, in stage 3, the
// z-slab [ny][nx][nz']; W1 holds the x-slab's Stolt / y-IFFT volume
// [ny][nx'][nz].
int sar_slab_setup(sar_plan *p) {
  const SarDeviceView &v = p->v;
  const int G = p->slab_world, nxl = v.nx / G, nzl = v.nz / G;
  p->tma_w1x = p->tma_w1z = p->tma_r1 = false;
  p->tm_r1_ptr = nullptr;
  if (v.force_plain) return SAR_OK;
  const uint32_t rows1 = v.ny < K4A_ROWS ? v.ny : K4A_ROWS, xr = v.nx < 256 ? v.nx : 256;
  p->tma_w1x = encode3d(&p->tm_w1x_mid, v.w1, v.nz, nxl, v.ny, KC, 1, rows1);
  p->tma_w1z = encode3d(&p->tm_w1z_rows, v.w0, nzl, v.nx, v.ny, KC, xr, 1);
  return SAR_OK;
}

int sar_slab_launch(sar_plan *p, int stage, const void *d_in, void *d_out, void *d_image, cudaStream_t s,
                    void *const *peers) {
  const SarDeviceView &v = p->v;
  const int G = p->slab_world, r = p->slab_rank;
  const int nxl = v.nx / G, nyl = v.ny / G, nzl = v.nz / G;
  const size_t c8 = sizeof(float2);
  cudaError_t e = cudaSuccess;
  if (stage == 1) {
    SarDeviceView vk = v;
    vk.vy0 = r * nyl;
    vk.nvy = nyl;
    // K1's epilogue stores every column straight into its destination block
    // (the packed send buffer, or slot `rank` of the peer's receive buffer)
    const long long hs1 = (long long)nyl * nxl * v.nk * c8;
    const BlockDst bd = peers ? dst_peers(peers, G, r, hs1) : dst_packed(d_out, G, hs1);
    int lg = 0;
    while ((1 << lg) < nxl) ++lg;
    vk.slab_lg = lg;
    for (int h = 0; h < G; ++h) vk.slab_dst[h] = reinterpret_cast<float2 *>(bd.d[h]);
    const CUtensorMap *tm_s = nullptr;
    if (p->tma_ap) {
      if (p->tm_s_ptr != d_in) p->tma_s = sar_encode_input_map(p, d_in);
      if (p->tma_s) tm_s = &p->tm_s;
    }
    SAR_CHECK(launch_k1(vk, static_cast<const float2 *>(d_in), true, s, tm_s, p->tma_ap ? &p->tm_ap : nullptr,
                        p->k1_br, p->k1_regacc, p->num_sms));
    return SAR_OK;
  }
  if (stage == 2) {
    float2 *xs = static_cast<float2 *>(const_cast<void *>(d_in));   // the x-slab [ny][nx'][nk], overwritten
    const CUtensorMap *tm = nullptr;
    if (!v.force_plain) {
      if (p->tm_r1_ptr != d_in) {
        const uint32_t rows = v.ny < 256 ? v.ny : 256;
        p->tma_r1 = encode3d(&p->tm_r1_mid, xs, v.nk, nxl, v.ny, KC, 1, rows);
        p->tm_r1_ptr = d_in;
      }
      if (p->tma_r1) tm = &p->tm_r1_mid;
    }
    const int *lbx = v.liveb ? v.liveb + r * nxl : nullptr;   // this x-slab's columns
    SAR_CHECK(launch_mid<-1>(xs, v.tw_y, 1, v.ny, nxl, v.nk, s, tm, p->num_sms, nullptr, lbx));
    SarDeviceView vk = v;
    vk.nx = nxl;
    vk.cls = p->d_slab_cls;
    vk.ncls = p->slab_ncls;
    vk.w0 = xs;
    vk.w0_elems = (size_t)v.ny * nxl * v.nk;   // the received x-slab (SAR_CHECKED bounds)
    SAR_CHECK(launch_k3(vk, true, s, p->num_sms));
    // y-IFFT; exchange #2 takes block h = z-slots [h nz', (h+1) nz') of every
    // column: stored there by the y-IFFT's own epilogue when a 16-wide z chunk
    // never straddles two blocks, else packed by a copy
    const long long hs2 = (long long)v.ny * nxl * nzl * c8;
    const BlockDst bd2 = peers ? dst_peers(peers, G, r, hs2) : dst_packed(d_out, G, hs2);
    if (p->tma_w1x && nzl % KC == 0 && v.ny <= 512) {
      MidSlabOut so{};
      so.nzl = nzl;
      for (int h = 0; h < G; ++h) so.d[h] = bd2.d[h];
      SAR_CHECK(launch_mid<+1>(v.w1, v.tw_y, 1, v.ny, nxl, v.nz, s, &p->tm_w1x_mid, p->num_sms, &so, lbx));
    } else {
      SAR_CHECK(launch_mid<+1>(v.w1, v.tw_y, 1, v.ny, nxl, v.nz, s, p->tma_w1x ? &p->tm_w1x_mid : nullptr,
                               p->num_sms, nullptr, lbx));
      SAR_CHECK(block_copy(bd2, v.w1, G, (long long)v.ny * nxl, (long long)nzl * c8, (long long)nzl * c8,
                           (long long)v.nz * c8, (long long)nzl * c8, p->num_sms, s));
    }
    return SAR_OK;
  }
  // stage 3: x-IFFT + magnitude of the received [G][ny][nx'][nz'] (block g =
  // columns [g nx', (g+1) nx')): read in place through a 4-D tensor map
  // (one box = one [nx][16] tile), or unpacked into the z-slab [ny][nx][nz']
  // (in W0) when the map does not apply
  if (!v.force_plain && nxl <= 256 && v.nx <= 512 && nzl % 2 == 0) {
    if (p->tm_r2_ptr != d_in) {
      p->tma_r2 = encode4d(&p->tm_r2_4d, d_in, nzl, nxl, v.ny, G, KC, nxl, 1, G);
      p->tm_r2_ptr = d_in;
    }
    if (p->tma_r2) {
      SarDeviceView vk = v;
      vk.nz = nzl;
      vk.z_off = r * nzl;
      vk.nz_img = v.nz;
      SAR_CHECK(launch_k4b(vk, d_image, (p->flags & SAR_OUTPUT_COMPLEX) != 0, s, &p->tm_r2_4d, p->num_sms, true));
      return SAR_OK;
    }
  }
  float2 *zs = v.w0;
  SAR_CHECK(block_copy(dst_packed(zs, G, (long long)nxl * nzl * c8), d_in, G, v.ny, (long long)nxl * nzl * c8,
                       (long long)v.ny * nxl * nzl * c8, (long long)nxl * nzl * c8, (long long)v.nx * nzl * c8,
                       p->num_sms, s));
  SarDeviceView vk = v;
  vk.nz = nzl;
  vk.z_off = r * nzl;
  vk.nz_img = v.nz;
  vk.w1 = zs;
  vk.w1_elems = v.w0_elems;
  SAR_CHECK(launch_k4b(vk, d_image, (p->flags & SAR_OUTPUT_COMPLEX) != 0, s, p->tma_w1z ? &p->tm_w1z_rows : nullptr,
                       p->num_sms));
  return SAR_OK;
}
