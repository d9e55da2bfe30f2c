// plan_internal.h -- the plan object shared by the host C ABI (plan.cpp) and
// the kernel launchers (pipeline.cu and the per-kernel translation units).
// Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sar_b200.h"

// rows per TMA box of the inverse y-FFT (K4a, fft_mid.cu): K4a reads only the
// boxes that hold live rows, so K3's class list covers whole boxes (plan.cpp)
#ifndef K4A_ROWS
#define K4A_ROWS 32
#endif

#define SAR_PROFILE_RING 1024
#define SAR_N_STAGES 5

// One Stolt mirror class (a, b), 0 <= a <= nx/2, 0 <= b <= ny/2: the up to 4
// spectral columns (+-a, +-b) that share k_r^2 (built on the host, plan.cpp).
struct SarClass {
  double kr2;      // k_x[a]^2 + k_y[b]^2 (IEEE, no contraction; reading R9)
  int jlo, jhi;    // superset of the in-band k_z bins (empty if jhi < jlo)
  int nmem, pad;   // member columns
  int col[4];      // column index b'*nx + a' of each member
};

// NUFFT spread (K1s) block of fine cells and its entry: one virtual element
// seen from one block (reading R19).
#define SAR_SP_BX 4
#define SAR_SP_BY 4
struct SarSpreadEntry {
  int row;      // sample row (f * npair + pair) * P + pose of the raw input
  float du, dv; // fine position relative to the block origin (unwrapped)
  float beta;   // -2 d_z + beta_MIMO (m); phase = beta * k
};

// SAR_GRID_NEAREST (reading R20): one (frame, pair, pose) sample row landing
// on a lattice node; the plan lists them per node (CSR) in (pair, pose) order.
struct SarNearEntry {
  int row;      // sample row (f * npair + pair) * P + pose of the raw input
  float beta;   // -2 d_z + beta_MIMO (m), the fp32 sum K1 forms; phase = beta * k
};

// Everything a kernel needs, passed by value (fits the 32 KB parameter space).
struct SarDeviceView {
  int F, nt, nr, npair, npx, npy, P, nk, nx, ny, nz;
  int f0;               // first frame of this launch (frame waves): raw rows, beta, R_ref and
                        // peak tables are indexed by f0 + f, the workspace by f
  int roll_x, roll_y;
  // slab decomposition (sar_slab_*; whole-image plans: 0, ny, (nx/2+1)(ny/2+1), 0, nz)
  int vy0, nvy;         // K1: virtual rows [vy0, vy0 + nvy) written as rows 0.. of w0
  int slab_lg;          // K1 slab epilogue: -1 off, else log2(nx'); column a of row vyl goes to
  float2 *slab_dst[SAR_MAX_SLAB];  //   slab_dst[a >> slab_lg] + (vyl nx' + a % nx') nk (packed or a peer)
  int ncls;             // K3: entries of cls
  int z_off, nz_img;    // K4b: the nz z-slots are z_off.. of an nz_img-plane image
  int zroll;            // output z roll: nz/2 (3-D, reading R8), 0 (2-D planes)
  int mode2d;           // SAR_IMAGE_2D: kz[] holds z_s - z_ref per plane (reading R18)
  int no_comp;
  int jx[SAR_MAX_PAIRS], jy[SAR_MAX_PAIRS];  // virtual-node offsets, pair = t*nr + r
  // SAR_GRID_NUFFT (reading R19): fine grid 2 nx x 2 ny, Gaussian half width
  // nu_w fine cells, variance nu_s2
  int nufft, nu_w;
  float nu_s2;
  const float *nu_decx, *nu_decy;  // [nx], [ny] 1/Phi deconvolution factors
  float2 *wh;                      // [F][2 ny][2 nx][nk] fine grid (spread, then x-transformed in place)
  int sp_nbx, sp_nby;              // spread blocks per fine row / column
  const int *sp_off;               // [F*sp_nby*sp_nbx + 1] CSR offsets
  const SarSpreadEntry *sp_ent;    // entries
  const float2 *tw_f;              // [2 nx] exp(-2 pi i m / (2 nx)) (fine x-FFT)
  int stolt_nufft;                 // SAR_STOLT_NUFFT (reading R21)
  const float *sn_dec;             // [nz] 1/Phi(m) of the depth in storage slot m mod nz
  int nearest;                     // SAR_GRID_NEAREST
  const int *nn_off;               // [F*ny*nx + 1] CSR offsets per lattice node (frame, vy, vx)
  const SarNearEntry *nn_ent;      // entries
  const float *apose;   // [F][P]      -2 d_z (m), fp32
  const float *bpair;   // [F][npair]  (d_x^2+d_y^2)/(4 R_ref) (m), fp32
  const float *kturn;   // [nk]        k_i / (2 pi) (turns per metre), fp32
  const double *k;      // [nk]        k_i (rad/m)
  const double *kx;     // [nx]
  const double *ky;     // [ny]
  const double *kz;     // [nz]        uniform Stolt grid (reading R5)
  const double *rref;   // [F]         R_ref = z_ref - Z_0
  const SarClass *cls;  // [ncls] the mirror classes K3 computes (those with a non-zero column,
                        // DESIGN.md section 6; all classes when liveb == nullptr)
  const int *liveb;     // [nx] live rows |b_s| <= liveb[a] of spectral column a (-1: none), or
                        // nullptr: every column is computed
  const float2 *pinv;   // [nk] 1/P(f) or nullptr (P == 1)
  const float2 *tw_x;   // [nx] exp(-2 pi i m/nx)
  const float2 *tw_y;   // [ny]
  const float2 *tw_z;   // [nz]
  const float2 *tw_z2;  // [2 nz] (SAR_STOLT_NUFFT fine grid)
  double k0, dk, inv_dk;
  double kz_top, kz_step;  // k_z[nz-1] = 2 k_max and the k_z bin width (reading R5)
  double stolt_delta;   // decision guard band of the fast Stolt path (common.cuh)
  int k1_step_ok;       // max |dk * beta| <= 0.25: K1 may use the Taylor step phasor
  int force_plain;      // SAR_FORCE_PLAIN: the plain (non-TMA, non-persistent) kernels
  float img_scale;      // 1/(nx ny nz)
  unsigned *peak;       // [F] max |voxel| bits per frame (SAR_REPORT_PEAK) or nullptr
  size_t w0_elems, w1_elems, raw_rows, img_elems;   // buffer sizes (SAR_CHECKED builds; img_elems 0: unchecked)
  float2 *w0;           // [F][ny][nx][nk]  planar lattice -> spectrum
  float2 *w1;           // [F][ny][nx][nz]  Stolt output -> partial inverse
};

struct sar_plan {
  // sizes
  int F = 0, nt = 0, nr = 0, npair = 0, npx = 0, npy = 0, P = 0, nk = 0, nx = 0, ny = 0, nz = 0;
  int wave = 0;   // frames per launch wave (= F without waves); the workspace holds `wave` frames
  uint32_t flags = 0;
  int device = 0;
  double dx = 0, dy = 0, dz = 0, z_ref = 0;
  double axes[6] = {0, 0, 0, 0, 0, 0};
  std::vector<int> jx, jy;
  std::vector<int32_t> col_range;   // [ny][nx][2] K3's in-band bin range of each column ({0,-1}: skipped)
  int jx_min = 0, jy_min = 0, nvx = 0, nvy = 0;
  SarDeviceView v{};
  // device allocations
  void *d_tables = nullptr;
  float2 *d_w0 = nullptr, *d_w1 = nullptr;
  size_t ws_bytes = 0;
  // host-buffer staging (sar_reconstruct_host)
  void *d_in = nullptr, *d_img = nullptr;
  size_t in_bytes = 0, img_bytes = 0;
  // profiling
  cudaEvent_t ev[SAR_PROFILE_RING][SAR_N_STAGES + 1];
  int n_prof = 0, n_prof_calls = 0;
  bool prof_events = false;
  cudaStream_t last_stream = nullptr;
  // TMA tensor maps over the workspace (built once per plan; valid flags)
  CUtensorMap tm_w0_mid, tm_w1_mid, tm_w1_rows, tm_ap, tm_s, tm_fine;
  bool tma_mid0 = false, tma_mid1 = false, tma_rows1 = false, tma_ap = false, tma_s = false, tma_fine = false;
  const void *tm_s_ptr = nullptr;  // data pointer tm_s was encoded for
  int k1_br = 0;                   // pose rows per K1 TMA box
  bool k1_regacc = false;          // every j^x offset is 0: K1 sums in registers
  int num_sms = 148;
  // SAR_CUDA_GRAPH: the recorded call and the (data, image) pair it was recorded for
  cudaStream_t cap_stream = nullptr;
  void *graph_exec = nullptr;   // CUgraphExec
  const void *g_data = nullptr;
  void *g_image = nullptr;
  // slab decomposition (sar_slab_create_slab); slab_world == 0: whole image
  int slab_rank = 0, slab_world = 0;
  SarClass *d_slab_cls = nullptr;
  int slab_ncls = 0;
  CUtensorMap tm_w1x_mid, tm_w1z_rows, tm_r1_mid, tm_r2_4d;
  bool tma_w1x = false, tma_w1z = false, tma_r1 = false, tma_r2 = false;
  const void *tm_r1_ptr = nullptr, *tm_r2_ptr = nullptr;
  // NUFFT mode tables and the half-transformed fine grid
  void *d_nu = nullptr;
  unsigned *d_peak = nullptr;   // SAR_REPORT_PEAK

  float2 *d_wh = nullptr;
};

// pipeline.cu
// SAR_CUDA_GRAPH: record the whole call (all frame waves) on p->cap_stream and
// launch it on s
int sar_graph_reconstruct(sar_plan *p, const void *d_data, void *d_image, cudaStream_t s);
// plan.cpp: the launches of one call (all frame waves) on s
int sar_enqueue_call(sar_plan *p, const void *d_data, void *d_image, cudaStream_t s);
void sar_graph_destroy(sar_plan *p);
int sar_launch_pipeline(sar_plan *p, const void *d_data, void *d_image, cudaStream_t s,
                        int stop_stage /*0 = full*/, int complex_out, cudaEvent_t *ev /*6 or null*/, int f0,
                        int nf);
int sar_launch_stolt_index(sar_plan *p, const int32_t *d_cols, int n, int32_t *d_i0, float *d_tau,
                           cudaStream_t s);
void sar_set_error(const std::string &msg);
int sar_build_tensor_maps(sar_plan *p);
int sar_slab_setup(sar_plan *p);
int sar_slab_launch(sar_plan *p, int stage, const void *d_in, void *d_out, void *d_image, cudaStream_t s,
                    void *const *peers = nullptr);
bool sar_encode_input_map(sar_plan *p, const void *d_data);
