// plan.cpp -- host side of the C ABI (include/sar_b200.h): argument
// validation, the fp64 geometry decomposition of Eqs. (3), (4), (7), (12)
// (P:123-153), table upload, workspace ownership, stage profiling.
// Compiled with -ffp-contract=off so that every table entry is the same IEEE
// expression the oracle evaluates (k_x, k_y, k_z, dk feed the bit-exact Stolt
// index decisions, reading R9).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "plan_internal.h"

#ifndef SAR_WAVE_BYTES
#define SAR_WAVE_BYTES 0   // L2 budget of one frame wave's W0 + W1; 0: no waves (measured slower)
#endif

namespace {
thread_local std::string g_last_error;

bool pow2_in_range(int n) { return n >= 2 && n <= SAR_MAX_FFT && (n & (n - 1)) == 0; }

int fail(int status, const std::string &msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char *what) {
  g_last_error = std::string("CUDA: ") + cudaGetErrorString(e) + " (" + what + ")";
  return SAR_ERR_CUDA;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void free_plan(sar_plan *p) {
  if (!p) return;
  DeviceGuard g(p->device);
  // the plan's work was enqueued on last_stream (NULL = the legacy default
  // stream, whose synchronisation is what that stream promises)
  cudaStreamSynchronize(p->last_stream);
  sar_graph_destroy(p);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  if (p->prof_events)
    for (int i = 0; i < SAR_PROFILE_RING; ++i)
      for (int j = 0; j <= SAR_N_STAGES; ++j) cudaEventDestroy(p->ev[i][j]);
  cudaFree(p->d_tables);
  cudaFree(p->d_w0);
  cudaFree(p->d_w1);
  cudaFree(p->d_in);
  cudaFree(p->d_img);
  cudaFree(p->d_wh);
  cudaFree(p->d_peak);
  cudaFree(p->d_slab_cls);
  delete p;
}

// twiddle table exp(-2 pi i m / n), fp64 -> fp32
void twiddles(std::vector<float> &dst, int n) {
  for (int m = 0; m < n; ++m) {
    const double a = -2.0 * M_PI * (double)m / (double)n;
    dst.push_back((float)cos(a));
    dst.push_back((float)sin(a));
  }
}
}  // namespace

void sar_set_error(const std::string &msg) { g_last_error = msg; }

extern "C" {

const char *sar_last_error(void) { return g_last_error.c_str(); }

int sar_version(void) { return SAR_B200_VERSION; }

const char *sar_status_string(int s) {
  switch (s) {
    case SAR_OK: return "SAR_OK";
    case SAR_ERR_INVALID_ARG: return "SAR_ERR_INVALID_ARG";
    case SAR_ERR_GEOMETRY: return "SAR_ERR_GEOMETRY";
    case SAR_ERR_UNSUPPORTED: return "SAR_ERR_UNSUPPORTED";
    case SAR_ERR_OOM: return "SAR_ERR_OOM";
    case SAR_ERR_CUDA: return "SAR_ERR_CUDA";
    default: return "SAR_ERR_UNKNOWN";
  }
}

}  // extern "C"

namespace {

// Host tables produced by the fp64 decomposition (uploaded by sar_plan_create).
struct HostTables {
  std::vector<float> apose, bpair, kturn, pinv, tw;
  std::vector<SarClass> cls;
  // the classes K3 computes and the live-row bound of every spectral column
  // (empty liveb: every column is computed)
  std::vector<SarClass> live;
  std::vector<int> liveb;
  // NUFFT mode
  std::vector<float> nu_decx, nu_decy;
  // NUFFT spread blocks (K1s): CSR of entries per (frame, 4 x 8 fine-cell block)
  std::vector<int> sp_off;
  std::vector<SarSpreadEntry> sp_ent;
  // SAR_GRID_NEAREST: pose nodes [F*P] and the CSR of entries per lattice node
  std::vector<int32_t> nn_ix, nn_iy;
  std::vector<float> sn_dec;     // SAR_STOLT_NUFFT deconvolution table [nz]
  std::vector<int> nn_off;
  std::vector<SarNearEntry> nn_ent;
  int sp_nbx = 0, sp_nby = 0;
  size_t tw_f_off = 0;
  std::vector<double> kx, ky, kz, kd, rref;
  size_t tw_y_off = 0, tw_z_off = 0, tw_z2_off = 0;
  int roll_x = 0, roll_y = 0;
  double k0 = 0, dk = 0, dkz = 0;
};

// Validation + Eqs. (3),(4),(7),(12) decomposition, no device involved.
int host_decompose(const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags, sar_plan *p,
                   HostTables &T) {
  double &dkz = T.dkz;
  if (!g || !im) return fail(SAR_ERR_INVALID_ARG, "geometry or image descriptor is NULL");
  if (g->n_frames < 0) return fail(SAR_ERR_INVALID_ARG, "n_frames < 0");
  if (g->n_tx < 1 || g->n_rx < 1) return fail(SAR_ERR_INVALID_ARG, "n_tx and n_rx must be >= 1");
  if (g->n_tx * g->n_rx > SAR_MAX_PAIRS) return fail(SAR_ERR_UNSUPPORTED, "n_tx*n_rx > SAR_MAX_PAIRS");
  if (!g->tx_xyz || !g->rx_xyz || !g->k) return fail(SAR_ERR_INVALID_ARG, "tx_xyz, rx_xyz or k is NULL");
  if (g->n_frames > 0 && !g->scan_xyz) return fail(SAR_ERR_INVALID_ARG, "scan_xyz is NULL");
  if (g->npx < 1 || g->npy < 1) return fail(SAR_ERR_INVALID_ARG, "npx, npy must be >= 1");
  if (g->n_k < 2) return fail(SAR_ERR_INVALID_ARG, "n_k must be >= 2");
  if (g->n_k > SAR_MAX_NK) return fail(SAR_ERR_UNSUPPORTED, "n_k > SAR_MAX_NK");
  const bool mode2d = (flags & SAR_IMAGE_2D) != 0;
  if (!pow2_in_range(im->nx) || !pow2_in_range(im->ny))
    return fail(SAR_ERR_INVALID_ARG, "nx, ny must be powers of two in [2, SAR_MAX_FFT]");
  if (mode2d) {
    if (im->nz < 1 || im->nz > SAR_MAX_FFT) return fail(SAR_ERR_INVALID_ARG, "2-D plans need 1..SAR_MAX_FFT planes");
    if (!im->z_planes) return fail(SAR_ERR_INVALID_ARG, "SAR_IMAGE_2D needs z_planes");
  } else if (!pow2_in_range(im->nz)) {
    return fail(SAR_ERR_INVALID_ARG, "nz must be a power of two in [2, SAR_MAX_FFT]");
  }
  if (g->npx > im->nx || g->npy > im->ny) return fail(SAR_ERR_INVALID_ARG, "raster larger than the FFT grid");
  if ((flags & SAR_GRID_NUFFT) && (im->nx > 512 || im->ny > 512 || g->npx > 512 || im->nx < 32))
    return fail(SAR_ERR_UNSUPPORTED, "SAR_GRID_NUFFT needs 32 <= nx <= 512, ny <= 512, npx <= 512");
  if ((flags & SAR_GRID_NUFFT) && (flags & SAR_GRID_NEAREST))
    return fail(SAR_ERR_INVALID_ARG, "SAR_GRID_NEAREST and SAR_GRID_NUFFT are exclusive");
  if ((flags & SAR_STOLT_NUFFT) && mode2d)
    return fail(SAR_ERR_INVALID_ARG, "SAR_STOLT_NUFFT needs the 3-D k_z grid (not SAR_IMAGE_2D)");
  if ((flags & SAR_STOLT_NUFFT) && im->nz > 512) return fail(SAR_ERR_UNSUPPORTED, "SAR_STOLT_NUFFT needs nz <= 512");
  if (!(g->dx > 0) || !(g->dy > 0) || (!mode2d && !(im->dz > 0)))
    return fail(SAR_ERR_INVALID_ARG, "pitches must be > 0");
  // K1's TMA row coordinate and the NUFFT spread entries index raw sample rows
  // (frame, pair, pose) with 32-bit ints
  if ((long long)g->n_frames * g->n_tx * g->n_rx * g->npx * g->npy >= (1LL << 31))
    return fail(SAR_ERR_UNSUPPORTED, "n_frames * n_tx * n_rx * poses >= 2^31 sample rows");
  if (g->n_frames > 65535) return fail(SAR_ERR_UNSUPPORTED, "n_frames > 65535");

  const int F = g->n_frames, nt = g->n_tx, nr = g->n_rx, nk = g->n_k;
  const int P = g->npx * g->npy;
  // O0: uniform wavenumber grid
  T.k0 = g->k[0];
  T.dk = (g->k[nk - 1] - g->k[0]) / (double)(nk - 1);
  if (!(T.dk > 0)) return fail(SAR_ERR_GEOMETRY, "k must be ascending");
  for (int i = 0; i < nk; ++i)
    if (fabs(g->k[i] - (T.k0 + (double)i * T.dk)) > 1e-9 * T.k0) return fail(SAR_ERR_GEOMETRY, "k grid not uniform");

  p->F = F; p->nt = nt; p->nr = nr; p->npair = nt * nr; p->npx = g->npx; p->npy = g->npy; p->P = P;
  p->nk = nk; p->nx = im->nx; p->ny = im->ny; p->nz = im->nz; p->flags = flags; p->device = g->device;
  p->dx = g->dx; p->dy = g->dy; p->dz = im->dz; p->z_ref = im->z_ref;

  // Eq. (3): virtual element at the Tx/Rx midpoint; lattice offset j = rint(m/pitch)
  std::vector<double> bm(p->npair);
  p->jx.assign(p->npair, 0);
  p->jy.assign(p->npair, 0);
  const double mz = g->tx_xyz[2];
  for (int t = 0; t < nt; ++t)
    for (int r = 0; r < nr; ++r) {
      const double *tx = g->tx_xyz + 3 * t, *rx = g->rx_xyz + 3 * r;
      if (tx[2] != rx[2] || tx[2] != mz) return fail(SAR_ERR_GEOMETRY, "Tx and Rx must share one z plane (P:111)");
      const double mx = (tx[0] + rx[0]) / 2.0, my = (tx[1] + rx[1]) / 2.0;
      const double bx = rx[0] - tx[0], by = rx[1] - tx[1];
      const double fx = mx / g->dx, fy = my / g->dy;
      const double jxr = nearbyint(fx), jyr = nearbyint(fy);
      if (fabs(fx - jxr) > 1e-6 || fabs(fy - jyr) > 1e-6)
        return fail(SAR_ERR_GEOMETRY, "Tx/Rx midpoints are not on the virtual lattice");
      p->jx[t * nr + r] = (int)jxr;
      p->jy[t * nr + r] = (int)jyr;
      bm[t * nr + r] = bx * bx + by * by;
    }
  p->jx_min = *std::min_element(p->jx.begin(), p->jx.end());
  p->jy_min = *std::min_element(p->jy.begin(), p->jy.end());
  int jxmax = 0, jymax = 0;
  for (int i = 0; i < p->npair; ++i) {
    p->jx[i] -= p->jx_min;
    p->jy[i] -= p->jy_min;
    jxmax = std::max(jxmax, p->jx[i]);
    jymax = std::max(jymax, p->jy[i]);
  }
  p->nvx = p->npx + jxmax;
  p->nvy = p->npy + jymax;

  // Eq. (4): Z_0, R_ref and the per-pose beta term -2 d_z (reading R1)
  std::vector<double> z0(F);
  T.rref.assign(F, 0.0);
  for (int f = 0; f < F; ++f) {
    if (g->z0) {
      z0[f] = g->z0[f];
    } else {
      double acc = 0;
      for (int q = 0; q < P; ++q) acc += g->scan_xyz[((size_t)f * P + q) * 3 + 2];
      z0[f] = acc / (double)P;
    }
    T.rref[f] = im->z_ref - z0[f];
    if (!(T.rref[f] > 0)) return fail(SAR_ERR_GEOMETRY, "z_ref must lie beyond the reference plane (R_ref > 0)");
  }
  const bool nocomp = (flags & SAR_NO_COMPENSATION) != 0;
  T.apose.assign((size_t)F * P, 0.f);
  T.bpair.assign((size_t)F * p->npair, 0.f);
  for (int f = 0; f < F; ++f) {
    for (int q = 0; q < P; ++q) {
      const double dzp = g->scan_xyz[((size_t)f * P + q) * 3 + 2] + mz - z0[f];
      T.apose[(size_t)f * P + q] = nocomp ? 0.f : (float)(-2.0 * dzp);
    }
    for (int i = 0; i < p->npair; ++i)
      T.bpair[(size_t)f * p->npair + i] = nocomp ? 0.f : (float)(bm[i] / (4.0 * T.rref[f]));
  }
  // wavenumber tables (reading R2) and the k_z grid (reading R5)
  T.kx.resize(p->nx);
  T.ky.resize(p->ny);
  T.kz.resize(p->nz);
  T.kd.assign(g->k, g->k + nk);
  for (int a = 0; a < p->nx; ++a) {
    const int as = a < p->nx / 2 ? a : a - p->nx;
    T.kx[a] = 2.0 * M_PI * (double)as / ((double)p->nx * g->dx);
  }
  for (int b = 0; b < p->ny; ++b) {
    const int bs = b < p->ny / 2 ? b : b - p->ny;
    T.ky[b] = 2.0 * M_PI * (double)bs / ((double)p->ny * g->dy);
  }
  if (mode2d) {
    // 2-D plans: the "k_z table" holds the plane offsets z_s - z_ref (reading R18)
    dkz = 1.0;
    for (int j = 0; j < p->nz; ++j) T.kz[j] = im->z_planes[j] - im->z_ref;
  } else {
    dkz = 2.0 * M_PI / ((double)p->nz * im->dz);
    for (int j = 0; j < p->nz; ++j) T.kz[j] = 2.0 * g->k[nk - 1] - (double)(p->nz - 1 - j) * dkz;
  }
  T.kturn.resize(nk);
  for (int i = 0; i < nk; ++i) T.kturn[i] = (float)(g->k[i] / (2.0 * M_PI));
  T.pinv.clear();
  if (g->pulse) {
    for (int i = 0; i < nk; ++i) {
      const double re = g->pulse[2 * i], im_ = g->pulse[2 * i + 1];
      const double d = re * re + im_ * im_;
      if (!(d > 0)) return fail(SAR_ERR_INVALID_ARG, "pulse spectrum has a zero");
      T.pinv.push_back((float)(re / d));
      T.pinv.push_back((float)(-im_ / d));
    }
  }
  T.tw.clear();
  twiddles(T.tw, p->nx);
  T.tw_y_off = T.tw.size() / 2;
  twiddles(T.tw, p->ny);
  T.tw_z_off = T.tw.size() / 2;
  twiddles(T.tw, p->nz);
  T.tw_z2_off = T.tw.size() / 2;
  if (flags & SAR_STOLT_NUFFT) twiddles(T.tw, 2 * p->nz);   // the NUFFT Stolt fine grid

  // Stolt mirror classes: k_r^2, member columns and a superset of the in-band
  // k_z bins.  u(j) = (sqrt(k_z,j^2 + k_r^2)/2 - k_0)/dk is monotone in j; the
  // band edges u = 0 and u = n_k - 1 sit at k_z = sqrt(4 k_0^2 - k_r^2) and
  // sqrt(4 k_max^2 - k_r^2); the range is widened by 2 bins each side and to
  // the whole axis when an edge lies within 1e-3 bins of k_z = 0 (du/dj -> 0
  // there).  Bins outside are zero; the device's bit-exact pull decides inside.
  {
    const int hx = p->nx / 2 + 1, hy = p->ny / 2 + 1, nz = p->nz;
    const double kmax = T.k0 + (double)(nk - 1) * T.dk, kz_top = mode2d ? 2.0 * kmax : T.kz[nz - 1];
    T.cls.resize((size_t)hx * hy);
    for (int b = 0; b < hy; ++b)
      for (int a = 0; a < hx; ++a) {
        SarClass &c = T.cls[(size_t)b * hx + a];
        memset(&c, 0, sizeof(c));
        const double kxa = T.kx[a] * T.kx[a], kyb = T.ky[b] * T.ky[b];
        c.kr2 = kxa + kyb;
        const int ma = (p->nx - a) & (p->nx - 1), mb = (p->ny - b) & (p->ny - 1);
        const int c4[4] = {b * p->nx + a, b * p->nx + ma, mb * p->nx + a, mb * p->nx + ma};
        const bool ok4[4] = {true, ma != a, mb != b, ma != a && mb != b};
        for (int m = 0; m < 4; ++m)
          if (ok4[m]) c.col[c.nmem++] = c4[m];
        const double qhi = 4.0 * kmax * kmax - c.kr2, qlo = 4.0 * T.k0 * T.k0 - c.kr2;
        if (!(qhi > 0.0)) {
          c.jlo = 0;
          c.jhi = -1;
          continue;
        }
        const double kzhi = sqrt(qhi), kzlo = qlo > 0.0 ? sqrt(qlo) : 0.0;
        if (kzlo < 1e-3 * dkz || kzhi < 1e-3 * dkz) {
          c.jlo = 0;
          c.jhi = nz - 1;
          continue;
        }
        const double jl = (double)(nz - 1) - (kz_top - kzlo) / dkz;
        const double jh = (double)(nz - 1) - (kz_top - kzhi) / dkz;
        const int lo = (int)std::max(floor(jl) - 2.0, 0.0);
        const int hi = (int)std::min(ceil(jh) + 2.0, (double)(nz - 1));
        c.jlo = lo;
        c.jhi = hi < lo ? lo - 1 : hi;
      }
  }

  // Columns whose Stolt output is provably zero are skipped by K3 (not read,
  // not written), their rows are not stored by K2 and read as zero by K4a:
  // evanescent columns, k_r^2 >= 4 k_max^2, where H = 0 for every k_i (Eq. (13),
  // P:211; reading R4), and, in 3-D, columns none of whose k_z bins can be in
  // band (jhi < jlo: the band lies below the k_z window).  Both conditions grow
  // with k_r^2, so the live rows of column a are |b_s| <= liveb[a]; the table
  // is checked for that shape and the skip is dropped if it does not hold.
  {
    const int hx = p->nx / 2 + 1, hy = p->ny / 2 + 1;
    const double kmax = T.k0 + (double)(nk - 1) * T.dk;
    auto dead = [&](const SarClass &c) {
      const double qhi = 4.0 * kmax * kmax - c.kr2;
      return !(qhi > 0.0) || (!mode2d && c.jhi < c.jlo);
    };
    std::vector<int> lb(p->nx, -1);
    for (int b = 0; b < hy; ++b)
      for (int a = 0; a < hx; ++a) {
        const SarClass &c = T.cls[(size_t)b * hx + a];
        if (dead(c)) continue;
        for (int m = 0; m < c.nmem; ++m) {
          const int ca = c.col[m] % p->nx;
          lb[ca] = std::max(lb[ca], b);
        }
      }
    bool shaped = true;
    for (int b = 0; b < hy; ++b)
      for (int a = 0; a < hx; ++a) {
        const SarClass &c = T.cls[(size_t)b * hx + a];
        if ((b <= lb[a]) == dead(c)) shaped = false;
      }
    // K4a reads whole boxes of R rows (those with a live row, the others are
    // zero-filled), so K3 also writes every row of those boxes: the classes it
    // computes are |b_s| <= lbk[a] (the extra ones are dead: zero output)
    const int R = std::min(p->ny, K4A_ROWS), N = p->ny;
    std::vector<int> lbk(p->nx, -1);
    for (int a = 0; a < p->nx; ++a)
      for (int bx = 0; bx < N / R; ++bx) {
        const bool live = lb[a] >= 0 && (bx * R <= lb[a] || (bx + 1) * R - 1 >= N - lb[a]);
        if (!live) continue;
        for (int m = bx * R; m < (bx + 1) * R; ++m) lbk[a] = std::max(lbk[a], m <= N / 2 ? m : N - m);
      }
    T.live.clear();
    p->col_range.assign((size_t)p->ny * p->nx * 2, 0);
    for (int b = 0; b < hy; ++b)
      for (int a = 0; a < hx; ++a) {
        const SarClass &c = T.cls[(size_t)b * hx + a];
        const bool skip = shaped && b > lbk[a];
        if (!skip) T.live.push_back(c);
        for (int m = 0; m < c.nmem; ++m) {
          p->col_range[2 * (size_t)c.col[m]] = skip ? 0 : c.jlo;
          p->col_range[2 * (size_t)c.col[m] + 1] = skip ? -1 : c.jhi;
        }
      }
#ifdef SAR_EXPERIMENT_NO_SKIP
    shaped = false;   // A/B experiments only (scripts/ab_variants.py)
    T.live = T.cls;
    for (size_t i = 0; i < p->col_range.size(); i += 2) p->col_range[i] = 0, p->col_range[i + 1] = p->nz - 1;
#endif
    if (shaped) T.liveb = lb;
    else T.liveb.clear();
  }

  // NUFFT placement tables (reading R19; must match oracle/nufft.py): fine
  // grid 2N per axis, Gaussian of half width W = 6 fine cells, variance
  // s2 = W / (2 pi (1 - 1/(2 sigma))), deconvolution 1/Phi(a) with
  // Phi(a) = sqrt(2 pi s2) exp(-2 pi^2 s2 a^2 / R^2)
  if (flags & SAR_GRID_NUFFT) {
    const int W = 6, sig = 2;
    const double s2 = W / (2.0 * M_PI * (1.0 - 1.0 / (2.0 * sig)));
    const int Rx = sig * p->nx, Ry = sig * p->ny;
    auto dec = [&](int n, int R, std::vector<float> &o) {
      o.resize(n);
      for (int a = 0; a < n; ++a) {
        const double as = a < n / 2 ? a : a - n;
        o[a] = (float)(1.0 / (sqrt(2.0 * M_PI * s2) * exp(-2.0 * M_PI * M_PI * s2 * as * as / ((double)R * R))));
      }
    };
    dec(p->nx, Rx, T.nu_decx);
    dec(p->ny, Ry, T.nu_decy);

    // K1s spread entries: every virtual element (f, pair, pose) at the fine
    // position (U, V) = sig ((x - x0)/dx + j^x, (y - y0)/dy + j^y) of its true
    // in-plane position reaches the fine cells |j - U| <= W, |i - V| <= W
    // (mod R, reading R6); it is listed once per SP_BY x SP_BX block those
    // cells touch, with its position relative to the (unwrapped) block origin
    // and its compensation term beta = -2 d_z + beta_MIMO (m; phase k beta).
    T.sp_nbx = Rx / SAR_SP_BX;
    T.sp_nby = Ry / SAR_SP_BY;
    const int nbx = T.sp_nbx, nby = T.sp_nby;
    const size_t nblk = (size_t)F * nby * nbx;
    auto fdiv = [](long long a, long long b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
    auto wmod = [](long long a, long long b) { return (int)(((a % b) + b) % b); };
    T.sp_off.assign(nblk + 1, 0);
    for (int pass = 0; pass < 2; ++pass) {
      std::vector<int> fill;
      if (pass == 1) {
        for (size_t i = 0; i < nblk; ++i) T.sp_off[i + 1] += T.sp_off[i];
        T.sp_ent.resize((size_t)T.sp_off[nblk]);
        fill.assign(T.sp_off.begin(), T.sp_off.end() - 1);
      }
      for (int f = 0; f < F; ++f)
        for (int pr = 0; pr < p->npair; ++pr)
          for (int q = 0; q < P; ++q) {
            const double *sp = g->scan_xyz + ((size_t)f * P + q) * 3;
            const double U = sig * ((sp[0] - g->x0) / g->dx + p->jx[pr]);
            const double V = sig * ((sp[1] - g->y0) / g->dy + p->jy[pr]);
            const long long xlo = (long long)ceil(U - W - 1e-4), xhi = (long long)floor(U + W + 1e-4);
            const long long ylo = (long long)ceil(V - W - 1e-4), yhi = (long long)floor(V + W + 1e-4);
            const float b = T.apose[(size_t)f * P + q] + T.bpair[(size_t)f * p->npair + pr];
            for (long long byr = fdiv(ylo, SAR_SP_BY); byr <= fdiv(yhi, SAR_SP_BY); ++byr)
              for (long long bxr = fdiv(xlo, SAR_SP_BX); bxr <= fdiv(xhi, SAR_SP_BX); ++bxr) {
                const size_t blk = ((size_t)f * nby + wmod(byr, nby)) * nbx + wmod(bxr, nbx);
                if (pass == 0) {
                  ++T.sp_off[blk + 1];
                } else {
                  SarSpreadEntry &e = T.sp_ent[(size_t)fill[blk]++];
                  e.row = (int)(((size_t)f * p->npair + pr) * P + q);
                  e.du = (float)(U - (double)(bxr * SAR_SP_BX));
                  e.dv = (float)(V - (double)(byr * SAR_SP_BY));
                  e.beta = b;
                }
              }
          }
    }
    T.tw_f_off = T.tw.size() / 2;
    twiddles(T.tw, Rx);
  }

  // NEAREST placement (reading R20; must match oracle.nearest_nodes): pose
  // node (rint((x - x0)/dx), rint((y - y0)/dy)) in fp64 (division first,
  // round-half-even), then + j_tr modulo the FFT grid (reading R6); the
  // entries of a node in (pair, pose) order, so with every pose on its raster
  // node the summation order is K1's (pairs in order)
  T.nn_ix.clear();
  T.nn_iy.clear();
  if (F > 0) {
    T.nn_ix.resize((size_t)F * P);
    T.nn_iy.resize((size_t)F * P);
    for (size_t i = 0; i < (size_t)F * P; ++i) {
      const double *sp = g->scan_xyz + i * 3;
      const double fx = nearbyint((sp[0] - g->x0) / g->dx), fy = nearbyint((sp[1] - g->y0) / g->dy);
      if (!(fabs(fx) < 1e9 && fabs(fy) < 1e9))
        return fail(SAR_ERR_UNSUPPORTED, "a NEAREST pose node does not fit 32 bits");
      T.nn_ix[i] = (int32_t)fx;
      T.nn_iy[i] = (int32_t)fy;
    }
  }
  if ((flags & SAR_GRID_NEAREST) && F > 0) {
    const size_t nnode = (size_t)F * p->ny * p->nx;
    auto wmod = [](long long a, long long b) { return (int)(((a % b) + b) % b); };
    T.nn_off.assign(nnode + 1, 0);
    for (int pass = 0; pass < 2; ++pass) {
      std::vector<int> fill;
      if (pass == 1) {
        for (size_t i = 0; i < nnode; ++i) T.nn_off[i + 1] += T.nn_off[i];
        T.nn_ent.resize((size_t)T.nn_off[nnode]);
        fill.assign(T.nn_off.begin(), T.nn_off.end() - 1);
      }
      for (int f = 0; f < F; ++f)
        for (int pr = 0; pr < p->npair; ++pr)
          for (int q = 0; q < P; ++q) {
            const size_t i = (size_t)f * P + q;
            const int vx = wmod((long long)T.nn_ix[i] + p->jx[pr], p->nx);
            const int vy = wmod((long long)T.nn_iy[i] + p->jy[pr], p->ny);
            const size_t node = ((size_t)f * p->ny + vy) * p->nx + vx;
            if (pass == 0) {
              ++T.nn_off[node + 1];
            } else {
              SarNearEntry &e = T.nn_ent[(size_t)fill[node]++];
              e.row = (int)(((size_t)f * p->npair + pr) * P + q);
              e.beta = T.apose[i] + T.bpair[(size_t)f * p->npair + pr];
            }
          }
    }
  }

  // NUFFT Stolt (reading R21; must match oracle/stolt_nufft.py): fine grid
  // R = 2 nz, Gaussian of variance s2 = W / (2 pi (1 - 1/(2 sigma))), W = 6;
  // storage slot q holds the signed depth m = q (q < nz/2) or q - nz, whose
  // deconvolution is 1/Phi(m), Phi(m) = sqrt(2 pi s2) exp(-2 pi^2 s2 m^2 / R^2)
  T.sn_dec.clear();
  if (flags & SAR_STOLT_NUFFT) {
    const double s2 = 6.0 / (2.0 * M_PI * (1.0 - 1.0 / 4.0));
    const double R = 2.0 * p->nz;
    T.sn_dec.resize(p->nz);
    for (int qz = 0; qz < p->nz; ++qz) {
      const double m = qz < p->nz / 2 ? qz : qz - p->nz;
      T.sn_dec[qz] = (float)(1.0 / (sqrt(2.0 * M_PI * s2) * exp(-2.0 * M_PI * M_PI * s2 * m * m / (R * R))));
    }
  }

  // O7 rolls and axes (reading R8)
  T.roll_x = p->nvx / 2 - p->nx / 2;
  T.roll_y = p->nvy / 2 - p->ny / 2;
  p->axes[0] = g->x0 + (double)(p->jx_min + T.roll_x) * g->dx;
  p->axes[1] = g->y0 + (double)(p->jy_min + T.roll_y) * g->dy;
  p->axes[2] = mode2d ? im->z_planes[0] : im->z_ref - (double)(p->nz / 2) * im->dz;
  p->axes[3] = g->dx;
  p->axes[4] = g->dy;
  p->axes[5] = mode2d ? (p->nz > 1 ? im->z_planes[1] - im->z_planes[0] : 0.0) : im->dz;
  // Frame waves: a batch runs the five kernels on `wave` frames at a time, so
  // that a wave's intermediate volumes (W0 + W1) fit the L2 budget and the
  // kernel after the one that wrote them reads them from L2 (Realtime: 24 MiB
  // per frame).  The workspace holds one wave.
  {
    const size_t per_frame = (size_t)p->ny * p->nx * ((size_t)nk + p->nz) * sizeof(float2);
    int w = F;
    if (F > 1 && !(flags & SAR_GRID_NUFFT) && (size_t)SAR_WAVE_BYTES > 0) {
      const size_t fit = (size_t)SAR_WAVE_BYTES / per_frame;
      w = (int)std::min<size_t>((size_t)F, std::max<size_t>(1, fit));
    }
    p->wave = w;
  }
  // W0 [wave][ny][nx][nk] + W1 [wave][ny][nx][nz] (+ the NUFFT fine grid [F][2ny][2nx][nk])
  p->ws_bytes = ((size_t)p->wave * p->ny * p->nx * ((size_t)nk + p->nz) +
                 ((flags & SAR_GRID_NUFFT) ? (size_t)F * p->ny * p->nx * 4 * (size_t)nk : 0)) *
                sizeof(float2);
  return SAR_OK;
}

}  // namespace

extern "C" {

int sar_plan_describe(const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags, sar_plan_info *info,
                      int32_t *jx, int32_t *jy, double *kx, double *ky, double *kz, float *apose, float *bpair) {
  if (!info) return fail(SAR_ERR_INVALID_ARG, "info is NULL");
  sar_plan tmp;
  HostTables T;
  int st = host_decompose(g, im, flags, &tmp, T);
  if (st != SAR_OK) return st;
  info->n_pairs = tmp.npair;
  info->jx_min = tmp.jx_min;
  info->jy_min = tmp.jy_min;
  info->nvx = tmp.nvx;
  info->nvy = tmp.nvy;
  info->roll_x = T.roll_x;
  info->roll_y = T.roll_y;
  memcpy(info->axes, tmp.axes, sizeof(tmp.axes));
  info->k0 = T.k0;
  info->dk = T.dk;
  info->workspace_bytes = tmp.ws_bytes;
  for (int i = 0; i < tmp.npair; ++i) {
    if (jx) jx[i] = tmp.jx[i];
    if (jy) jy[i] = tmp.jy[i];
  }
  if (kx) memcpy(kx, T.kx.data(), T.kx.size() * sizeof(double));
  if (ky) memcpy(ky, T.ky.data(), T.ky.size() * sizeof(double));
  if (kz) memcpy(kz, T.kz.data(), T.kz.size() * sizeof(double));
  if (apose) memcpy(apose, T.apose.data(), T.apose.size() * sizeof(float));
  if (bpair) memcpy(bpair, T.bpair.data(), T.bpair.size() * sizeof(float));
  return SAR_OK;
}

}  // extern "C"

namespace {
// slab_world > 0: the plan of one rank of a slab decomposition, whose
// workspace holds only the slab volumes: W1 = the x-slab [ny][nx/G][nz] and
// W0 = the z-slab [ny][nx][nz/G] (the stage-3 unpack target)
int plan_create_impl(sar_plan **out, const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags,
                     int slab_world) {
  if (!out) return fail(SAR_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  sar_plan *p = new (std::nothrow) sar_plan();
  if (!p) return fail(SAR_ERR_OOM, "host allocation failed");
  HostTables T;
  int st = host_decompose(g, im, flags, p, T);
  if (st != SAR_OK) {
    delete p;
    return st;
  }
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0) {
    delete p;
    return fail(SAR_ERR_UNSUPPORTED, "no CUDA device");
  }
  if (g->device < 0 || g->device >= ndev) {
    delete p;
    return fail(SAR_ERR_INVALID_ARG, "device ordinal out of range");
  }
  cudaDeviceProp prop;
  ce = cudaGetDeviceProperties(&prop, g->device);
  if (ce != cudaSuccess) {
    delete p;
    return cuda_fail(ce, "cudaGetDeviceProperties");
  }
  if (prop.major != 10 || prop.minor != 0) {
    delete p;
    return fail(SAR_ERR_UNSUPPORTED, "this build targets sm_100a (B200) only; device is sm_" +
                                         std::to_string(prop.major) + std::to_string(prop.minor));
  }
  const int F = p->F, nk = p->nk, P = p->P;

  // one device allocation for all tables (256-byte aligned sections)
  DeviceGuard guard(p->device);
  auto al = [](size_t n) { return (n + 255) & ~(size_t)255; };
  size_t off = 0;
  const size_t o_ap = off; off += al(T.apose.size() * 4);
  const size_t o_bp = off; off += al(T.bpair.size() * 4);
  const size_t o_kt = off; off += al(T.kturn.size() * 4);
  const size_t o_k = off; off += al(T.kd.size() * 8);
  const size_t o_kx = off; off += al(T.kx.size() * 8);
  const size_t o_ky = off; off += al(T.ky.size() * 8);
  const size_t o_kz = off; off += al(T.kz.size() * 8);
  const size_t o_rr = off; off += al(T.rref.size() * 8 + 8);
  const size_t o_pi = off; off += al(T.pinv.size() * 4);
  const size_t o_tw = off; off += al(T.tw.size() * 4);
  const size_t o_cl = off; off += al(T.live.size() * sizeof(SarClass));
  const size_t o_lb = off; off += al(T.liveb.size() * 4);
  const size_t o_nu_dx = off; off += al(T.nu_decx.size() * 4);
  const size_t o_nu_dy = off; off += al(T.nu_decy.size() * 4);
  const size_t o_sp_off = off; off += al(T.sp_off.size() * 4);
  const size_t o_sp_ent = off; off += al(T.sp_ent.size() * sizeof(SarSpreadEntry));
  const size_t o_nn_off = off; off += al(T.nn_off.size() * 4);
  const size_t o_sn = off; off += al(T.sn_dec.size() * 4);
  const size_t o_nn_ent = off; off += al(T.nn_ent.size() * sizeof(SarNearEntry));
  ce = cudaMalloc(&p->d_tables, off);
  if (ce != cudaSuccess) {
    cudaGetLastError();
    free_plan(p);
    return fail(SAR_ERR_OOM, "table allocation failed");
  }
  char *base = (char *)p->d_tables;
  auto up = [&](size_t o, const void *src, size_t n) {
    return n ? cudaMemcpy(base + o, src, n, cudaMemcpyHostToDevice) : cudaSuccess;
  };
  if ((ce = up(o_ap, T.apose.data(), T.apose.size() * 4)) != cudaSuccess ||
      (ce = up(o_bp, T.bpair.data(), T.bpair.size() * 4)) != cudaSuccess ||
      (ce = up(o_kt, T.kturn.data(), T.kturn.size() * 4)) != cudaSuccess ||
      (ce = up(o_k, T.kd.data(), T.kd.size() * 8)) != cudaSuccess ||
      (ce = up(o_kx, T.kx.data(), T.kx.size() * 8)) != cudaSuccess ||
      (ce = up(o_ky, T.ky.data(), T.ky.size() * 8)) != cudaSuccess ||
      (ce = up(o_kz, T.kz.data(), T.kz.size() * 8)) != cudaSuccess ||
      (ce = up(o_rr, T.rref.data(), T.rref.size() * 8)) != cudaSuccess ||
      (ce = up(o_pi, T.pinv.data(), T.pinv.size() * 4)) != cudaSuccess ||
      (ce = up(o_tw, T.tw.data(), T.tw.size() * 4)) != cudaSuccess ||
      (ce = up(o_cl, T.live.data(), T.live.size() * sizeof(SarClass))) != cudaSuccess ||
      (ce = up(o_lb, T.liveb.data(), T.liveb.size() * 4)) != cudaSuccess ||
      (ce = up(o_nu_dx, T.nu_decx.data(), T.nu_decx.size() * 4)) != cudaSuccess ||
      (ce = up(o_nu_dy, T.nu_decy.data(), T.nu_decy.size() * 4)) != cudaSuccess ||
      (ce = up(o_sp_off, T.sp_off.data(), T.sp_off.size() * 4)) != cudaSuccess ||
      (ce = up(o_sp_ent, T.sp_ent.data(), T.sp_ent.size() * sizeof(SarSpreadEntry))) != cudaSuccess ||
      (ce = up(o_nn_off, T.nn_off.data(), T.nn_off.size() * 4)) != cudaSuccess ||
      (ce = up(o_sn, T.sn_dec.data(), T.sn_dec.size() * 4)) != cudaSuccess ||
      (ce = up(o_nn_ent, T.nn_ent.data(), T.nn_ent.size() * sizeof(SarNearEntry))) != cudaSuccess) {
    free_plan(p);
    return cuda_fail(ce, "table upload");
  }
  size_t n0 = (size_t)p->wave * p->ny * p->nx * nk, n1 = (size_t)p->wave * p->ny * p->nx * p->nz;
  if (slab_world > 0) {
    n0 = n1 = (size_t)p->ny * p->nx * (p->nz / slab_world);
    p->ws_bytes = (n0 + n1) * sizeof(float2);
    p->slab_world = slab_world;
  }
  if (F > 0) {
    if (cudaMalloc(&p->d_w0, n0 * sizeof(float2)) != cudaSuccess ||
        cudaMalloc(&p->d_w1, n1 * sizeof(float2)) != cudaSuccess ||
      ((flags & SAR_GRID_NUFFT) && cudaMalloc(&p->d_wh, 4 * (size_t)F * p->ny * p->nx * nk * sizeof(float2)) != cudaSuccess)) {
      cudaGetLastError();
      free_plan(p);
      return fail(SAR_ERR_OOM, "workspace allocation failed");
    }
  }
  SarDeviceView &v = p->v;
  v.F = F; v.f0 = 0; v.nt = p->nt; v.nr = p->nr; v.npair = p->npair; v.npx = p->npx; v.npy = p->npy; v.P = P;
  v.nk = nk; v.nx = p->nx; v.ny = p->ny; v.nz = p->nz;
  v.roll_x = T.roll_x; v.roll_y = T.roll_y;
  v.no_comp = (flags & SAR_NO_COMPENSATION) ? 1 : 0;
  for (int i = 0; i < p->npair; ++i) {
    v.jx[i] = p->jx[i] % p->nx;  // placement mod the FFT grid (reading R6)
    v.jy[i] = p->jy[i] % p->ny;
  }
  v.apose = (const float *)(base + o_ap);
  v.bpair = (const float *)(base + o_bp);
  v.kturn = (const float *)(base + o_kt);
  v.k = (const double *)(base + o_k);
  v.kx = (const double *)(base + o_kx);
  v.ky = (const double *)(base + o_ky);
  v.kz = (const double *)(base + o_kz);
  v.rref = (const double *)(base + o_rr);
  v.nufft = (flags & SAR_GRID_NUFFT) ? 1 : 0;
  v.nu_w = 6;
  v.nu_s2 = (float)(6.0 / (2.0 * M_PI * (1.0 - 1.0 / 4.0)));
  v.nu_decx = (const float *)(base + o_nu_dx);
  v.nu_decy = (const float *)(base + o_nu_dy);
  v.sp_nbx = T.sp_nbx;
  v.sp_nby = T.sp_nby;
  v.sp_off = (const int *)(base + o_sp_off);
  v.sp_ent = (const SarSpreadEntry *)(base + o_sp_ent);
  v.tw_f = (const float2 *)(base + o_tw) + T.tw_f_off;
  v.nearest = (flags & SAR_GRID_NEAREST) ? 1 : 0;
  v.stolt_nufft = (flags & SAR_STOLT_NUFFT) ? 1 : 0;
  v.sn_dec = (const float *)(base + o_sn);
  v.nn_off = (const int *)(base + o_nn_off);
  v.nn_ent = (const SarNearEntry *)(base + o_nn_ent);
  v.cls = (const SarClass *)(base + o_cl);
  v.liveb = T.liveb.empty() ? nullptr : (const int *)(base + o_lb);
  v.pinv = T.pinv.empty() ? nullptr : (const float2 *)(base + o_pi);
  v.tw_x = (const float2 *)(base + o_tw);
  v.tw_y = (const float2 *)(base + o_tw) + T.tw_y_off;
  v.tw_z = (const float2 *)(base + o_tw) + T.tw_z_off;
  v.tw_z2 = (const float2 *)(base + o_tw) + T.tw_z2_off;
  v.k0 = T.k0;
  v.dk = T.dk;
  v.inv_dk = 1.0 / T.dk;
  v.kz_top = T.kz.back();
  v.kz_step = T.dkz;
  {
    // |u_fast - u| <= (2e-13 * kk + 4 ulp(u)) / dk with kk <= k_max (fast_dsqrt bound)
    const double kmax = T.kd.back();
    const double err = (2e-13 * kmax) / T.dk + 4.0 * 2.220446049250313e-16 * (double)nk;
    v.stolt_delta = std::max(1e-7, 100.0 * err);
  }
  v.mode2d = (flags & SAR_IMAGE_2D) ? 1 : 0;
  v.zroll = v.mode2d ? 0 : p->nz / 2;
  v.vy0 = 0;
  v.nvy = p->ny;
  v.slab_lg = -1;
  v.ncls = (int)T.live.size();
  v.z_off = 0;
  v.nz_img = p->nz;
  v.img_scale = (float)(1.0 / ((double)p->nx * p->ny * (v.mode2d ? 1 : p->nz)));
  {
    // K1 step phasor exp(j dk beta): 5th-order Taylor needs |dk beta| small
    float amax = 0.f, bmax = 0.f;
    for (float a : T.apose) amax = std::max(amax, fabsf(a));
    for (float b : T.bpair) bmax = std::max(bmax, fabsf(b));
    v.k1_step_ok = (T.dk * ((double)amax + (double)bmax) <= 0.25) ? 1 : 0;
  }
  if ((flags & SAR_REPORT_PEAK) && F > 0) {
    if (cudaMalloc(&p->d_peak, (size_t)F * sizeof(unsigned)) != cudaSuccess) {
      cudaGetLastError();
      free_plan(p);
      return fail(SAR_ERR_OOM, "peak buffer allocation failed");
    }
  }
  v.peak = p->d_peak;
  v.w0 = p->d_w0;
  v.wh = p->d_wh;
  v.force_plain = (flags & SAR_FORCE_PLAIN) ? 1 : 0;
  v.w1 = p->d_w1;
  v.w0_elems = n0;
  v.w1_elems = n1;
  v.raw_rows = (size_t)F * p->npair * P;
  v.img_elems = slab_world > 0 ? 0 : (size_t)F * p->nz * p->ny * p->nx;

  p->num_sms = prop.multiProcessorCount;
#ifdef SAR_SM_LIMIT   // A/B builds: persistent grids on fewer SMs (sustained-load power experiments)
  if (p->num_sms > SAR_SM_LIMIT) p->num_sms = SAR_SM_LIMIT;
#endif
  sar_build_tensor_maps(p);
  if (flags & SAR_CUDA_GRAPH) {
    if (cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
      cudaGetLastError();
      free_plan(p);
      return fail(SAR_ERR_CUDA, "capture stream creation failed");
    }
  }
  if (flags & SAR_PROFILE_STAGES) {
    for (int i = 0; i < SAR_PROFILE_RING; ++i)
      for (int j = 0; j <= SAR_N_STAGES; ++j) cudaEventCreate(&p->ev[i][j]);
    p->prof_events = true;
  }
  *out = p;
  return SAR_OK;
}
}  // namespace

extern "C" {

int sar_plan_create(sar_plan **out, const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags) {
  return plan_create_impl(out, g, im, flags, 0);
}

int sar_plan_describe_stolt_ranges(const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags,
                                   int32_t *ranges) {
  if (!ranges) return fail(SAR_ERR_INVALID_ARG, "ranges is NULL");
  sar_plan tmp;
  HostTables T;
  int st = host_decompose(g, im, flags, &tmp, T);
  if (st != SAR_OK) return st;
  memcpy(ranges, tmp.col_range.data(), tmp.col_range.size() * sizeof(int32_t));
  return SAR_OK;
}

int sar_plan_describe_nearest(const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags, int32_t *ix,
                              int32_t *iy) {
  if (!ix || !iy) return fail(SAR_ERR_INVALID_ARG, "ix or iy is NULL");
  sar_plan tmp;
  HostTables T;
  int st = host_decompose(g, im, flags & ~(uint32_t)SAR_GRID_NEAREST, &tmp, T);
  if (st != SAR_OK) return st;
  if (!T.nn_ix.empty()) {
    memcpy(ix, T.nn_ix.data(), T.nn_ix.size() * sizeof(int32_t));
    memcpy(iy, T.nn_iy.data(), T.nn_iy.size() * sizeof(int32_t));
  }
  return SAR_OK;
}

int sar_plan_create_slab(sar_plan **out, const sar_geom_desc *g, const sar_image_desc *im, uint32_t flags,
                         const sar_slab_desc *slab) {
  if (!out) return fail(SAR_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!slab || !g || !im) return fail(SAR_ERR_INVALID_ARG, "slab, geometry or image descriptor is NULL");
  const int G = slab->world, r = slab->rank;
  if (G < 1 || G > SAR_MAX_SLAB || r < 0 || r >= G) return fail(SAR_ERR_INVALID_ARG, "slab rank/world out of range");
  if (flags & (SAR_IMAGE_2D | SAR_GRID_NUFFT | SAR_GRID_NEAREST | SAR_STOLT_NUFFT | SAR_REPORT_PEAK | SAR_CUDA_GRAPH))
    return fail(SAR_ERR_UNSUPPORTED, "slab plans support the 3-D RASTER path only");
  if (g->n_frames != 1) return fail(SAR_ERR_INVALID_ARG, "slab plans reconstruct one image (n_frames == 1)");
  if (im->nx % G || im->ny % G || im->nz % G || im->nx / G < 1 || im->nz / G < 1)
    return fail(SAR_ERR_INVALID_ARG, "world must divide nx, ny and nz");
  sar_plan *p = nullptr;
  int st = plan_create_impl(&p, g, im, flags, G);
  if (st != SAR_OK) return st;
  DeviceGuard guard(p->device);
  p->slab_rank = r;
  // the x-slab's Stolt classes: every mirror class restricted to the member
  // columns a in [r nx', (r+1) nx'), local column index b nx' + (a - r nx');
  // k_r^2 and the in-band range are the whole-image class's (bit-identical)
  const int nxl = p->nx / G, a0 = r * nxl;
  std::vector<SarClass> full((size_t)p->v.ncls), mine;
  cudaError_t ce = cudaMemcpy(full.data(), p->v.cls, full.size() * sizeof(SarClass), cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) {
    sar_plan_destroy(p);
    return cuda_fail(ce, "class table download");
  }
  for (const SarClass &c : full) {
    SarClass m = c;
    m.nmem = 0;
    for (int i = 0; i < c.nmem; ++i) {
      const int b = c.col[i] / p->nx, a = c.col[i] - b * p->nx;
      if (a >= a0 && a < a0 + nxl) m.col[m.nmem++] = b * nxl + (a - a0);
    }
    if (m.nmem) mine.push_back(m);
  }
  p->slab_ncls = (int)mine.size();
  if (cudaMalloc(&p->d_slab_cls, std::max<size_t>(1, mine.size()) * sizeof(SarClass)) != cudaSuccess) {
    cudaGetLastError();
    sar_plan_destroy(p);
    return fail(SAR_ERR_OOM, "slab class table allocation failed");
  }
  ce = cudaMemcpy(p->d_slab_cls, mine.data(), mine.size() * sizeof(SarClass), cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) {
    sar_plan_destroy(p);
    return cuda_fail(ce, "slab class table upload");
  }
  st = sar_slab_setup(p);
  if (st != SAR_OK) {
    sar_plan_destroy(p);
    return st;
  }
  *out = p;
  return SAR_OK;
}

int sar_slab_buffer_bytes(const sar_plan *p, size_t *send1, size_t *send2) {
  if (!p || !send1 || !send2) return fail(SAR_ERR_INVALID_ARG, "NULL argument");
  if (p->slab_world < 1) return fail(SAR_ERR_INVALID_ARG, "not a slab plan");
  const int G = p->slab_world;
  *send1 = (size_t)(p->ny / G) * p->nx * p->nk * sizeof(float) * 2;
  *send2 = (size_t)p->ny * (p->nx / G) * p->nz * sizeof(float) * 2;
  return SAR_OK;
}

int sar_slab_stage(sar_plan *p, int32_t stage, const void *d_in, void *d_out, void *d_image, sar_stream stream) {
  if (!p) return fail(SAR_ERR_INVALID_ARG, "plan is NULL");
  if (p->slab_world < 1) return fail(SAR_ERR_INVALID_ARG, "not a slab plan");
  if (stage < 1 || stage > 3) return fail(SAR_ERR_INVALID_ARG, "stage must be 1, 2 or 3");
  if (!d_in || (stage < 3 && !d_out) || (stage == 3 && !d_image))
    return fail(SAR_ERR_INVALID_ARG, "NULL buffer");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  p->last_stream = s;
  return sar_slab_launch(p, stage, d_in, d_out, d_image, s);
}

int sar_slab_stage_peers(sar_plan *p, int32_t stage, const void *d_in, void *const *peer_recv, sar_stream stream) {
  if (!p) return fail(SAR_ERR_INVALID_ARG, "plan is NULL");
  if (p->slab_world < 1) return fail(SAR_ERR_INVALID_ARG, "not a slab plan");
  if (stage != 1 && stage != 2) return fail(SAR_ERR_INVALID_ARG, "peer stores exist for stages 1 and 2");
  if (!d_in || !peer_recv) return fail(SAR_ERR_INVALID_ARG, "NULL buffer");
  for (int h = 0; h < p->slab_world; ++h)
    if (!peer_recv[h]) return fail(SAR_ERR_INVALID_ARG, "NULL peer buffer");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  p->last_stream = s;
  return sar_slab_launch(p, stage, d_in, nullptr, nullptr, s, peer_recv);
}

}  // extern "C"

// the launches of one call (all frame waves) on s
int sar_enqueue_call(sar_plan *p, const void *d_data, void *d_image, cudaStream_t s) {
  const int cplx = (p->flags & SAR_OUTPUT_COMPLEX) ? 1 : 0;
  if (p->d_peak) {
    cudaError_t e = cudaMemsetAsync(p->d_peak, 0, (size_t)p->F * sizeof(unsigned), s);
    if (e != cudaSuccess) return cuda_fail(e, "peak reset");
  }
  const size_t frame_img = (size_t)p->nz * p->ny * p->nx * (cplx ? sizeof(float2) : sizeof(float));
  for (int f0 = 0; f0 < p->F; f0 += p->wave) {
    const int st = sar_launch_pipeline(p, d_data, static_cast<char *>(d_image) + (size_t)f0 * frame_img, s, 0, cplx,
                                       nullptr, f0, std::min(p->wave, p->F - f0));
    if (st != SAR_OK) return st;
  }
  return SAR_OK;
}

extern "C" {

int sar_reconstruct(sar_plan *p, const void *d_data, void *d_image, sar_stream stream) {
  if (!p) return fail(SAR_ERR_INVALID_ARG, "plan is NULL");
  if (p->slab_world) return fail(SAR_ERR_INVALID_ARG, "slab plans run sar_slab_stage");
  if (p->F == 0) return SAR_OK;
  if (!d_data || !d_image) return fail(SAR_ERR_INVALID_ARG, "data or image pointer is NULL");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  p->last_stream = s;
  if ((p->flags & SAR_CUDA_GRAPH) && !p->prof_events) return sar_graph_reconstruct(p, d_data, d_image, s);
  const int cplx = (p->flags & SAR_OUTPUT_COMPLEX) ? 1 : 0;
  if (p->d_peak) {
    cudaError_t e = cudaMemsetAsync(p->d_peak, 0, (size_t)p->F * sizeof(unsigned), s);
    if (e != cudaSuccess) return cuda_fail(e, "peak reset");
  }
  const size_t frame_img = (size_t)p->nz * p->ny * p->nx * (cplx ? sizeof(float2) : sizeof(float));
  if (p->prof_events) ++p->n_prof_calls;
  for (int f0 = 0; f0 < p->F; f0 += p->wave) {
    cudaEvent_t *ev = nullptr;
    if (p->prof_events && p->n_prof < SAR_PROFILE_RING) ev = p->ev[p->n_prof++];
    const int st = sar_launch_pipeline(p, d_data, static_cast<char *>(d_image) + (size_t)f0 * frame_img, s, 0, cplx,
                                       ev, f0, std::min(p->wave, p->F - f0));
    if (st != SAR_OK) return st;
  }
  return SAR_OK;
}

int sar_reconstruct_host(sar_plan *p, const void *h_data, void *h_image, sar_stream stream) {
  if (!p) return fail(SAR_ERR_INVALID_ARG, "plan is NULL");
  if (p->slab_world) return fail(SAR_ERR_INVALID_ARG, "slab plans run sar_slab_stage");
  if (p->F == 0) return SAR_OK;
  if (!h_data || !h_image) return fail(SAR_ERR_INVALID_ARG, "data or image pointer is NULL");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t in_b = (size_t)p->F * p->npair * p->P * p->nk * sizeof(float2);
  const size_t img_b = (size_t)p->F * p->nz * p->ny * p->nx *
                       ((p->flags & SAR_OUTPUT_COMPLEX) ? sizeof(float2) : sizeof(float));
  if (!p->d_in || !p->d_img) {
    // both staging buffers or neither (a failed call leaves no half state)
    cudaFree(p->d_in);
    cudaFree(p->d_img);
    p->d_in = p->d_img = nullptr;
    if (cudaMalloc(&p->d_in, in_b) != cudaSuccess || cudaMalloc(&p->d_img, img_b) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(p->d_in);
      cudaFree(p->d_img);
      p->d_in = p->d_img = nullptr;
      return fail(SAR_ERR_OOM, "staging allocation failed");
    }
    p->in_bytes = in_b;
    p->img_bytes = img_b;
  }
  cudaError_t e = cudaMemcpyAsync(p->d_in, h_data, in_b, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D");
  int st = sar_reconstruct(p, p->d_in, p->d_img, stream);
  if (st != SAR_OK) return st;
  e = cudaMemcpyAsync(h_image, p->d_img, img_b, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(e, "D2H");
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "synchronize");
  return SAR_OK;
}

int sar_plan_destroy(sar_plan *p) {
  free_plan(p);
  return SAR_OK;
}

int sar_plan_get_axes(const sar_plan *p, double out[6]) {
  if (!p || !out) return fail(SAR_ERR_INVALID_ARG, "NULL argument");
  memcpy(out, p->axes, sizeof(p->axes));
  return SAR_OK;
}

int sar_plan_peaks(sar_plan *p, float *h_peaks) {
  if (!p || !h_peaks) return fail(SAR_ERR_INVALID_ARG, "NULL argument");
  if (!p->d_peak) return fail(SAR_ERR_INVALID_ARG, "plan was created without SAR_REPORT_PEAK");
  DeviceGuard g(p->device);
  cudaError_t e = cudaStreamSynchronize(p->last_stream);
  if (e == cudaSuccess) e = cudaMemcpy(h_peaks, p->d_peak, (size_t)p->F * sizeof(float), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "peaks");
  return SAR_OK;
}

int sar_plan_workspace_bytes(const sar_plan *p, size_t *bytes) {
  if (!p || !bytes) return fail(SAR_ERR_INVALID_ARG, "NULL argument");
  *bytes = p->ws_bytes;
  return SAR_OK;
}

int sar_plan_launches_per_call(const sar_plan *p, int32_t *n) {
  if (!p || !n) return fail(SAR_ERR_INVALID_ARG, "NULL argument");
  // K1 (or the NUFFT spread + fine x-FFT + K2n), K2, K3, K4a, K4b
  *n = p->F > 0 ? ((p->flags & SAR_GRID_NUFFT) ? SAR_N_STAGES + 1 : SAR_N_STAGES) : 0;
  return SAR_OK;
}

int sar_plan_profile_reset(sar_plan *p) {
  if (!p) return fail(SAR_ERR_INVALID_ARG, "plan is NULL");
  p->n_prof = p->n_prof_calls = 0;
  return SAR_OK;
}

int sar_plan_profile_read(sar_plan *p, float ms_out[5], int32_t *n_calls) {
  if (!p || !ms_out) return fail(SAR_ERR_INVALID_ARG, "NULL argument");
  if (!p->prof_events) return fail(SAR_ERR_INVALID_ARG, "plan was created without SAR_PROFILE_STAGES");
  DeviceGuard g(p->device);
  for (int j = 0; j < SAR_N_STAGES; ++j) ms_out[j] = 0.f;
  for (int i = 0; i < p->n_prof; ++i) {
    cudaError_t e = cudaEventSynchronize(p->ev[i][SAR_N_STAGES]);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
    for (int j = 0; j < SAR_N_STAGES; ++j) {
      float ms = 0.f;
      e = cudaEventElapsedTime(&ms, p->ev[i][j], p->ev[i][j + 1]);
      if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
      ms_out[j] += ms;
    }
  }
  if (n_calls) *n_calls = p->n_prof_calls;
  return SAR_OK;
}

int sar_debug_stage(sar_plan *p, int32_t stage, const void *d_data, void *d_out, sar_stream stream) {
  if (!p) return fail(SAR_ERR_INVALID_ARG, "plan is NULL");
  if (stage < 1 || stage > 4) return fail(SAR_ERR_INVALID_ARG, "stage must be 1..4");
  if (stage == 1 && (p->flags & SAR_GRID_NUFFT)) return fail(SAR_ERR_INVALID_ARG, "no planar lattice in NUFFT mode");
  if (stage == 3 && (p->flags & SAR_STOLT_NUFFT))
    return fail(SAR_ERR_INVALID_ARG, "no uniform k_z grid with SAR_STOLT_NUFFT (debug stage 3)");
  if (p->slab_world) return fail(SAR_ERR_INVALID_ARG, "slab plans run sar_slab_stage");
  if (p->F == 0) return SAR_OK;
  if (!d_data || !d_out) return fail(SAR_ERR_INVALID_ARG, "NULL pointer");
  DeviceGuard g(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  p->last_stream = s;
  // wave by wave; each wave's stage result is copied out of the workspace
  const size_t fr = (size_t)p->ny * p->nx * (stage == 3 ? p->nz : stage == 4 ? p->nz : p->nk);
  for (int f0 = 0; f0 < p->F; f0 += p->wave) {
    const int nf = std::min(p->wave, p->F - f0);
    if (stage == 4) {
      const int st = sar_launch_pipeline(p, d_data, static_cast<float2 *>(d_out) + (size_t)f0 * fr, s, 0, 1, nullptr,
                                         f0, nf);
      if (st != SAR_OK) return st;
      continue;
    }
    const int st = sar_launch_pipeline(p, d_data, nullptr, s, stage, 0, nullptr, f0, nf);
    if (st != SAR_OK) return st;
    cudaError_t e = cudaMemcpyAsync(static_cast<float2 *>(d_out) + (size_t)f0 * fr, stage == 3 ? p->d_w1 : p->d_w0,
                                    (size_t)nf * fr * sizeof(float2), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "stage copy");
  }
  return SAR_OK;
}

int sar_debug_node_offsets(const sar_plan *p, int32_t *jx, int32_t *jy, int32_t *jx_min, int32_t *jy_min) {
  if (!p || !jx || !jy) return fail(SAR_ERR_INVALID_ARG, "NULL argument");
  for (int i = 0; i < p->npair; ++i) {
    jx[i] = p->jx[i];
    jy[i] = p->jy[i];
  }
  if (jx_min) *jx_min = p->jx_min;
  if (jy_min) *jy_min = p->jy_min;
  return SAR_OK;
}

int sar_debug_stolt_index(sar_plan *p, const int32_t *d_cols, int32_t n, int32_t *d_i0, float *d_tau,
                          sar_stream stream) {
  if (!p || n < 0 || (n > 0 && (!d_cols || !d_i0 || !d_tau))) return fail(SAR_ERR_INVALID_ARG, "bad argument");
  DeviceGuard g(p->device);
  return sar_launch_stolt_index(p, d_cols, n, d_i0, d_tau, (cudaStream_t)stream);
}

}  // extern "C"
