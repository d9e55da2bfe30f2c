/*
 * sar_b200.h -- C ABI of the B200-native reconstruction path of
 * arXiv 2305.02064 ("efficient near-field MIMO-SAR imaging for irregular
 * scanning geometries").  Citation keys: P:n = PAPER.md line n.
 *
 * The library reconstructs a 3-D reflectivity image o(x,y,z) from multistatic,
 * multi-planar frequency-domain samples s[f][tx][rx][pos][k] in four steps
 * (Fig. 3):
 *   1. multistatic->monostatic / multi-planar->planar phase correction
 *      s_hat = s * exp(+j k beta) (Eqs. (11)-(12)) accumulated on
 *      the virtual planar lambda/4 lattice (Eqs. (3)-(4));
 *   2. forward 2-D spatial FFT (FT_2D of Eq. (14));
 *   3. RMA filter k_z/P(f) e^{-j k_z Z0} and Stolt resampling onto a uniform
 *      k_z grid (Eqs. (13)-(14));
 *   4. inverse 3-D FFT and magnitude (IFT_3D of Eq. (14)).
 * Readings where the paper is silent are DESIGN.md section 3 (R1..R17).
 *
 * Conventions (all entry points):
 *  - Every function returns an int status (enum sar_status); nothing throws
 *    across the ABI.  On failure sar_last_error() returns a thread-local
 *    human-readable message.
 *  - "device pointer" = CUDA global memory on the plan's device; "host
 *    pointer" = ordinary (preferably pinned) host memory.
 *  - Array layouts are C order (last index fastest); complex64 is interleaved
 *    (re, im) float32.
 *  - Asynchronous CUDA faults surface as SAR_ERR_CUDA on a later call.
 */
#ifndef SAR_B200_H
#define SAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAR_B200_VERSION 6

typedef struct sar_plan sar_plan;       /* opaque */
typedef struct CUstream_st *sar_stream; /* == cudaStream_t; NULL = legacy default stream */

enum sar_status {
  SAR_OK = 0,
  SAR_ERR_INVALID_ARG = 1, /* null pointer, bad size, not a power of two, ... */
  SAR_ERR_GEOMETRY = 2,    /* non-uniform k, off-lattice Tx/Rx midpoint, R_ref <= 0, Tx/Rx planes differ */
  SAR_ERR_UNSUPPORTED = 3, /* device is not sm_100 (B200), size above the compiled limits */
  SAR_ERR_OOM = 4,         /* device allocation failed */
  SAR_ERR_CUDA = 5         /* a CUDA runtime error (launch, copy, asynchronous fault) */
};

enum sar_flags {
  SAR_NO_COMPENSATION = 1u << 0, /* beta == 0: plain RMA on the raw samples (the paper's
                                    failure baseline) */
  SAR_OUTPUT_COMPLEX = 1u << 1,  /* image is complex64 o (scaled, rolled) instead of |o| */
  SAR_PROFILE_STAGES = 1u << 2,  /* record CUDA events around every kernel (sar_plan_profile_read) */
  SAR_IMAGE_2D = 1u << 3         /* 2-D single-plane images (reading R18, "2-D Proposed" of Table I,
                                    P:394): step 3 becomes the back-propagation of every
                                    filtered column to each plane of sar_image_desc.z_planes summed
                                    over k (no Stolt), the image is [F][nz planes][ny][nx] */,
  SAR_REPORT_PEAK = 1u << 5,     /* every call also records max |image| of each frame on the device
                                    (sar_plan_peaks); the normalisation of the eps_inf metric and of
                                    display (reading R11) without another pass over the image */
  SAR_GRID_NUFFT = 1u << 4       /* NUFFT placement (reading R19; FGG-NUFFT of P:239-242): steps 1-2
                                    become a type-1 non-uniform transform of the compensated samples
                                    from their TRUE (x', y') positions (fast Gaussian gridding,
                                    oversampling 2, half width 6 fine cells) instead of the RASTER
                                    lattice + FFT.  Needs nx <= 512, npx <= 512; debug stage 1 is
                                    not available (there is no lattice).  Combines with
                                    SAR_IMAGE_2D (NUFFT spectrum, then the plane sums) */,
  SAR_FORCE_PLAIN = 1u << 6,     /* testing: run the plain (non-TMA, non-persistent) kernel of every
                                    stage instead of the TMA-pipelined ones; same arithmetic, results
                                    equal to fp32 rounding (the coverage of the fallback kernels) */
  SAR_GRID_NEAREST = 1u << 8,    /* NEAREST placement (reading R20): step 1 puts every
                                    pose on the lambda/4 lattice node NEAREST its true in-plane
                                    position, (ix, iy) = (rint((x - x0)/dx), rint((y - y0)/dy)) in
                                    fp64, instead of its raster index (RASTER, reading R7); poses
                                    that land on one node are summed, nodes no pose reaches are 0,
                                    placement is modulo the FFT grid (reading R6).  The in-plane
                                    error is then <= pitch/2 instead of the jitter (the paper's
                                    FGG-NUFFT treatment of P:239-242 is SAR_GRID_NUFFT).  Not with
                                    SAR_GRID_NUFFT (INVALID_ARG) or slab plans (UNSUPPORTED) */
  SAR_STOLT_NUFFT = 1u << 9,     /* NUFFT Stolt step (reading R21; "NUFFT ... for the Fourier
                                    transforms and Stolt interpolation step"): step 3
                                    takes every filtered column along z from its non-uniform
                                    k_z,i = sqrt(4 k_i^2 - k_r^2) by a 1-D type-1 NUFFT (fast
                                    Gaussian gridding, oversampling 2, half width 6; samples
                                    weighted by the Jacobian 4 k_i dk / (k_z,i dk_z)) instead of
                                    the linear pull onto the uniform k_z grid and the z-IFFT.
                                    3-D only (INVALID_ARG with SAR_IMAGE_2D), nz <= 512
                                    (UNSUPPORTED); debug stage 3 is not available */
  SAR_CUDA_GRAPH = 1u << 7       /* replay the call's launches as one CUDA graph (for small, launch-bound
                                    configurations): the first sar_reconstruct with a given
                                    (d_data, d_image) pair records the path into a graph on a stream of
                                    the plan's own, later calls with the same pair launch that graph on
                                    the caller's stream (a new pair re-records); same kernels, same
                                    results.  Not combined with SAR_PROFILE_STAGES */
};

/* Limits of this build. */
#define SAR_MAX_FFT 1024  /* nx, ny, nz <= 1024 (powers of two >= 2) */
#define SAR_MAX_PAIRS 64  /* n_tx * n_rx <= 64 */
#define SAR_MAX_NK 2048   /* n_k <= 2048 (a Stolt column must fit in shared memory) */

/* Acquisition geometry (host memory; copied by sar_plan_create, so the caller
 * may free every array as soon as the call returns). */
typedef struct {
  int32_t n_frames;        /* F >= 0 independent frames (F = 0: every call is a no-op) */
  int32_t n_tx, n_rx;      /* >= 1 each, n_tx*n_rx <= SAR_MAX_PAIRS */
  const double *tx_xyz;    /* [n_tx][3] Tx positions in the radar body frame (m) */
  const double *rx_xyz;    /* [n_rx][3] Rx positions in the radar body frame (m); tx.z == rx.z */
  int32_t npx, npy;        /* nominal raster: pose p = iy*npx + ix, 1 <= npx <= nx, 1 <= npy <= ny */
  double x0, y0;           /* nominal world position of pose (0,0) (m); only the output axes use it */
  double dx, dy;           /* raster = virtual-lattice pitch (m), lambda/4 in the paper */
  const double *scan_xyz;  /* [F][npy*npx][3] actual radar positions, world frame (m); the z
                              coordinate gives the plane displacement d_z (Eq. (4)); x,y are
                              not used in RASTER placement (reading R7), they are the
                              non-uniform positions of SAR_GRID_NUFFT (reading R19) */
  const double *z0;        /* [F] reference plane Z_0 per frame (m), or NULL = mean of scan z */
  int32_t n_k;             /* 2 <= n_k <= SAR_MAX_NK frequency samples */
  const double *k;         /* [n_k] wavenumbers 2*pi*f/c (rad/m), uniform (1e-9 rel.), ascending */
  const double *pulse;     /* [n_k][2] complex P(f) (re,im) or NULL for P == 1 (Eq. (14)) */
  int32_t device;          /* CUDA device ordinal */
} sar_geom_desc;

/* Image grid. */
typedef struct {
  int32_t nx, ny;  /* spatial FFT size = image x/y size; powers of two in [2, SAR_MAX_FFT] */
  int32_t nz;      /* Stolt bins = image z size; power of two in [2, SAR_MAX_FFT].
                      With SAR_IMAGE_2D: the number of planes, 1..SAR_MAX_FFT (any count) */
  double dz;       /* image z pitch (m); k_z grid spacing 2*pi/(nz*dz) (reading R5); unused in 2-D */
  double z_ref;    /* reference depth (m): centre of the z window and R_ref = z_ref - Z_0 > 0 */
  const double *z_planes; /* SAR_IMAGE_2D only: [nz] plane depths z_s (world, m; host memory, copied);
                             ignored (may be NULL) otherwise */
} sar_image_desc;

/* Host-side result of the geometry decomposition (no device needed). */
typedef struct {
  int32_t n_pairs;           /* n_tx * n_rx */
  int32_t jx_min, jy_min;    /* minima of rint(midpoint/pitch) over the pairs (subtracted) */
  int32_t nvx, nvy;          /* virtual aperture extent in nodes: npx + max jx, npy + max jy */
  int32_t roll_x, roll_y;    /* output rolls floor(nv/2) - n/2 (reading R8) */
  double axes[6];            /* as sar_plan_get_axes */
  double k0, dk;             /* k[0] and (k[n_k-1]-k[0])/(n_k-1) */
  size_t workspace_bytes;    /* device workspace a plan would allocate */
} sar_plan_info;

/* Validate and decompose a geometry on the host only (no CUDA device is
 * touched): the same checks and fp64 tables sar_plan_create computes.  Any
 * of the optional outputs may be NULL; sizes: jx, jy [n_tx*n_rx] (offsets
 * after min-subtraction, row-major [n_tx][n_rx]); kx [nx], ky [ny], kz [nz]
 * (rad/m, the tables the Stolt step uses); apose [F*P] (-2 d_z, float32) and
 * bpair [F*n_tx*n_rx] ((d_x^2+d_y^2)/(4 R_ref), float32), both zero with
 * SAR_NO_COMPENSATION.  Errors: INVALID_ARG, GEOMETRY, UNSUPPORTED. */
int sar_plan_describe(const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags,
                      sar_plan_info *info, int32_t *jx, int32_t *jy, double *kx, double *ky,
                      double *kz, float *apose, float *bpair);

/* Host-only export of the Stolt bin range step 3 computes for every spectral
 * column (Eqs. (13)-(14); readings R5, R9): ranges[(b*nx + a)*2]
 * = jlo, [+1] = jhi, a superset of the k_z bins j whose pull can be in band
 * (the bit-exact fp64 decision runs only there, every other bin is zero).
 * jhi < jlo marks a column with no bin in band, whose Stolt output is zero:
 * evanescent (k_r^2 >= 4 k_max^2) or its band below the k_z window; the plan
 * skips such columns (no read, no write) except where the inverse y-FFT reads
 * them as part of a 32-row box.  ranges: host int32 [ny][nx][2].  Errors: as
 * sar_plan_describe. */
int sar_plan_describe_stolt_ranges(const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags,
                                   int32_t *ranges);

/* Host-only export of the SAR_GRID_NEAREST pose nodes (reading R20):
 * ix[f*P + p] = rint((x - x0)/dx), iy[f*P + p] = rint((y - y0)/dy) of pose p
 * of frame f (fp64, round-half-even; before the pair offsets j_tr and the
 * modulo of the FFT grid).  ix, iy: host int32 [F*npy*npx].  The same table
 * step 1 uses when SAR_GRID_NEAREST is set (flags need not include it).
 * Errors: as sar_plan_describe; UNSUPPORTED if a node does not fit 32 bits. */
int sar_plan_describe_nearest(const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags,
                              int32_t *ix, int32_t *iy);

/* Create a plan: validates the geometry, runs the fp64 decomposition of
 * Eqs. (3),(4),(7),(12) on the host (virtual-node offsets j_tr, beta terms,
 * k_x/k_y/k_z tables), allocates the device workspace and uploads the tables.  *out receives the plan
 * (NULL on failure).  Errors: INVALID_ARG, GEOMETRY, UNSUPPORTED, OOM, CUDA. */
int sar_plan_create(sar_plan **out, const sar_geom_desc *g, const sar_image_desc *im,
                    uint32_t flags);
/* Workspace: F*ny*nx*(n_k+nz)*8 bytes (+ F*4*ny*nx*n_k*8 for the
 * SAR_GRID_NUFFT fine grid).  (A build with SAR_WAVE_BYTES > 0 processes a
 * batch W frames at a time with a W-frame workspace; measured slower.) */

/* Reconstruct (3-D volume, or the planes of a SAR_IMAGE_2D plan).
 * d_data: device, complex64 [F][n_tx][n_rx][npy*npx][n_k],
 * 8-byte aligned, read only, caller-owned.  d_image: device, float32
 * [F][nz][ny][nx] (complex64 with SAR_OUTPUT_COMPLEX), caller-owned, fully
 * overwritten.  Voxel (m,iy,ix) is at world (x_first+ix*dx, y_first+iy*dy,
 * z_first+m*dz), see sar_plan_get_axes.  Enqueues 5 kernels (6 with
 * SAR_GRID_NUFFT) on `stream` and returns without synchronising; no allocation.  Not re-entrant per plan (the
 * workspace is shared): use one plan per concurrent stream.
 * Each launch is wrapped in an NVTX range named after its stage (tools only).
 * Errors: INVALID_ARG (null pointers, a slab plan), CUDA. */
int sar_reconstruct(sar_plan *p, const void *d_data, void *d_image, sar_stream stream);

/* End-to-end variant with HOST buffers: copies h_data (same layout as d_data)
 * host->device, reconstructs, copies the image device->host and synchronises
 * `stream` before returning.  Device staging buffers are allocated on first
 * use and owned by the plan.  Pinned host memory gives full PCIe bandwidth.
 * Errors: INVALID_ARG, OOM, CUDA. */
int sar_reconstruct_host(sar_plan *p, const void *h_data, void *h_image, sar_stream stream);

/* Synchronise the plan's last stream and free everything.  NULL is a no-op. */
int sar_plan_destroy(sar_plan *p);

/* out[6] = {x_first, y_first, z_first, dx, dy, dz} of the output voxel grid
 * (each axis periodic with period n*pitch; reading R8).  2-D plans: z_first =
 * z_planes[0] and dz = z_planes[1] - z_planes[0] (0 for one plane). */
int sar_plan_get_axes(const sar_plan *p, double out[6]);

/* Bytes of device workspace owned by the plan (excluding staging buffers). */
int sar_plan_workspace_bytes(const sar_plan *p, size_t *bytes);

/* Stage profiling (plan created with SAR_PROFILE_STAGES): sum of the CUDA-event
 * durations (ms) of each of the 5 kernels over all calls since the last reset.
 * Synchronises the recorded events.  ms_out[5] = {K1 correct+x-FFT, K2 y-FFT,
 * K3 filter+Stolt+z-IFFT, K4a y-IFFT, K4b x-IFFT+magnitude}; *n_calls
 * receives the number of calls summed (at most 1024 since the last reset). */
int sar_plan_profile_read(sar_plan *p, float ms_out[5], int32_t *n_calls);
int sar_plan_profile_reset(sar_plan *p);

/* SAR_REPORT_PEAK plans: max |image voxel| of each frame of the last
 * sar_reconstruct call (after the 1/(nx ny nz) scaling).  Synchronises the
 * plan's last stream; h_peaks: host float[F].  Errors: INVALID_ARG (no flag,
 * NULL), CUDA. */
int sar_plan_peaks(sar_plan *p, float *h_peaks);

/* Number of kernel launches one sar_reconstruct call enqueues (5, 6 with
 * SAR_GRID_NUFFT; 0 if F = 0). */
int sar_plan_launches_per_call(const sar_plan *p, int32_t *n);

/* ---- single-image slab decomposition over G GPUs ----
 *
 * One image (F == 1) split over `world` = G ranks, one plan and one GPU per
 * rank; the caller moves the data between the three stages with two
 * all-to-all exchanges (e.g. NCCL all_to_all_single over NVLink).  With
 * nx' = nx/G, ny' = ny/G, nz' = nz/G (G must divide nx, ny and nz):
 *   stage 1 (rank r): K1 on the virtual rows [r ny', (r+1) ny') -- the
 *     correction + MIMO accumulation + x-FFT of those lattice rows (Eqs.
 *     (11)-(12); FT_2D along x) -- packed for exchange #1:
 *     d_out = complex64 [G][ny'][nx'][n_k], block h = the columns
 *     [h nx', (h+1) nx') destined for rank h.  d_in = the raw samples
 *     (the full [1][n_tx][n_rx][npy*npx][n_k] array; only the pose rows that
 *     reach this rank's lattice rows are read).
 *   exchange #1: rank h receives block h of every rank g in order of g:
 *     complex64 [G][ny'][nx'][n_k] == the x-slab [ny][nx'][n_k].
 *   stage 2 (rank r): on the x-slab (columns [r nx', (r+1) nx')): y-FFT (in
 *     place in d_in, which is overwritten), RMA filter + Stolt + z-IFFT
 *     (Eqs. (13)-(14)) and y-IFFT, packed for exchange #2:
 *     d_out = complex64 [G][ny][nx'][nz'], block h = the z-slots
 *     [h nz', (h+1) nz').
 *   exchange #2: rank h receives block h of every rank g in order of g:
 *     complex64 [G][ny][nx'][nz'].
 *   stage 3 (rank r): x-IFFT + magnitude of the z-slots [r nz', (r+1) nz']
 *     (d_in = the exchange-#2 receive buffer, read in place, not modified),
 *     written into d_image = float32 (complex64 with SAR_OUTPUT_COMPLEX)
 *     [nz][ny][nx], the same rolled layout as sar_reconstruct; only the nz'
 *     planes this rank owns are written (plane m = (z + nz/2) mod nz of
 *     z-slot z, reading R8), the others are left untouched.
 * Stages 1 and 2 store their blocks from the kernels' own epilogues (no
 * separate pack pass).  Every element is computed by the same arithmetic as
 * sar_reconstruct, so the assembled image equals the whole-image result bit
 * for bit.  All three
 * calls are asynchronous on `stream`; d_in / d_out / d_image are device
 * pointers owned by the caller, 16-byte aligned, and must not alias.  A slab
 * plan's workspace holds only its slabs (2 * ny*nx*nz/G*8 bytes), so it does
 * not run the whole-image entry points (sar_reconstruct, sar_reconstruct_host,
 * sar_debug_stage return INVALID_ARG). */
#define SAR_MAX_SLAB 16 /* world <= 16 */

typedef struct {
  int32_t rank;   /* 0 <= rank < world */
  int32_t world;  /* 1 <= G <= SAR_MAX_SLAB, divides nx, ny and nz */
} sar_slab_desc;

/* Create the plan of one rank.  Errors: as sar_plan_create, plus
 * INVALID_ARG (bad rank/world, G does not divide the sizes, F != 1) and
 * UNSUPPORTED (SAR_IMAGE_2D, SAR_GRID_NUFFT or SAR_REPORT_PEAK). */
int sar_plan_create_slab(sar_plan **out, const sar_geom_desc *g, const sar_image_desc *im,
                         uint32_t flags, const sar_slab_desc *slab);

/* Bytes of the stage-1 and stage-2 output buffers (= the exchange buffers):
 * *send1 = ny'*nx*n_k*8 (G blocks), *send2 = ny*nx'*nz*8 (G blocks).
 * Errors: INVALID_ARG (NULL, not a slab plan). */
int sar_slab_buffer_bytes(const sar_plan *p, size_t *send1, size_t *send2);

/* Run stage 1, 2 or 3 of this rank (see above).  Errors: INVALID_ARG (stage
 * outside 1..3, NULL pointers, not a slab plan), CUDA. */
int sar_slab_stage(sar_plan *p, int32_t stage, const void *d_in, void *d_out, void *d_image,
                   sar_stream stream);

/* Exchange by peer stores: stage 1 or 2 of this rank with the exchange
 * folded into its pack, so no all-to-all call is needed.  peer_recv: host
 * array of G device pointers, valid in this process (this GPU's own buffer
 * for h == rank, the others mapped from the peer GPUs, e.g. with CUDA IPC over
 * NVLink / NVSwitch), each rank h's receive buffer of the stage's exchange
 * (G blocks of sar_slab_buffer_bytes / G bytes); block h of this rank is
 * stored straight into slot `rank` of peer_recv[h].  The caller orders the
 * stages across ranks (e.g. stream sync + barrier) before the receivers read.
 * Stage 3 is sar_slab_stage.  Errors: INVALID_ARG (stage not 1 or 2, NULL),
 * CUDA. */
int sar_slab_stage_peers(sar_plan *p, int32_t stage, const void *d_in, void *const *peer_recv,
                         sar_stream stream);

/* ---- debug / parity entry points (same kernels as sar_reconstruct) ---- */

/* Run the path up to `stage` and copy that stage's result to d_out (device):
 *   1: planar lattice after correction, complex64 [F][ny][nx][n_k]
 *   2: spatial spectrum after the 2-D FFT, complex64 [F][ny][nx][n_k]
 *   3: Stolt output before the z-IFFT, complex64 [F][ny][nx][nz] (2-D plans:
 *      the plane spectra [F][ny][nx][n planes])
 *   4: rolled complex image, complex64 [F][nz][ny][nx] (scaled 1/(nx ny nz))
 * Errors: INVALID_ARG (stage outside 1..4, null pointers), CUDA. */
int sar_debug_stage(sar_plan *p, int32_t stage, const void *d_data, void *d_out,
                    sar_stream stream);

/* Host copies of the integer virtual-node offsets of every (tx,rx) pair after
 * min-subtraction (row-major [n_tx][n_rx]) and the minima subtracted. */
int sar_debug_node_offsets(const sar_plan *p, int32_t *jx, int32_t *jy, int32_t *jx_min,
                           int32_t *jy_min);

/* Stolt pull indices computed by the device code of step 3 for n columns
 * (d_cols: device int32 [n][2] = (a, b) spectral indices):
 * d_i0[n][nz] = floor index or -1 (zero bin), d_tau[n][nz] = weight (float32).
 * Errors: INVALID_ARG, CUDA. */
int sar_debug_stolt_index(sar_plan *p, const int32_t *d_cols, int32_t n, int32_t *d_i0,
                          float *d_tau, sar_stream stream);

/* ---- back-projection baseline (BPA) -------------------------
 *
 * The paper's gold standard and comparison system,
 * not a step of the reconstruction path: the matched filter of Eq. (9)
 * with the exact round-trip distances of Eq. (2) and
 * the ACTUAL element positions T_{t,p} = scan_xyz[p] + tx_xyz[t],
 * R_{r,p} = scan_xyz[p] + rx_xyz[r] (the radar keeps its orientation):
 *
 *   o(v) = sum_{t,r,p,i} s[t,r,p,i] exp(+j k_i (|v - T_{t,p}| + |v - R_{r,p}|))
 *
 * (no normalisation, no compensation, no lattice: every voxel costs
 * n_tx n_rx P n_k complex multiply-adds).  Of g only n_frames, n_tx, n_rx,
 * tx_xyz, rx_xyz, npx, npy, scan_xyz, n_k, k and device are read (k uniform
 * and ascending as for a plan; any positions).  frame: which frame of d_data.
 * d_data: device, complex64 [F][n_tx][n_rx][npy*npx][n_k] (the layout of
 * sar_reconstruct), read only.  h_voxels: HOST float64 [n_voxels][3] world
 * positions (m), copied.  d_out: device complex64 [n_voxels], overwritten.
 * ms_out: if not NULL receives the kernel's CUDA-event time (ms).  The call
 * allocates and frees its own device tables and SYNCHRONISES `stream` before
 * returning (a baseline, not a hot path).  n_voxels = 0 is a no-op.
 * Distances and phase reduction in fp64, the k loop in fp32 (DESIGN.md
 * section 10).  Errors: INVALID_ARG, GEOMETRY (k), UNSUPPORTED (not sm_100;
 * one pose's n_tx*n_rx*n_k samples above 200 KB), OOM, CUDA. */
int sar_bpa(const sar_geom_desc *g, int32_t frame, const void *d_data, const double *h_voxels,
            int64_t n_voxels, void *d_out, sar_stream stream, float *ms_out);

const char *sar_status_string(int status);
const char *sar_last_error(void);
int sar_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SAR_B200_H */
