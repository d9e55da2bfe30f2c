"""Thin ctypes binding of ``include/sar_b200.h`` (argument marshalling only).

Every step of the reconstruction runs in the CUDA library
``libsar_b200.so``; this module only converts NumPy/torch arguments to the C
ABI.  There is no CPU fallback: if the library is missing or the device is not
a B200 the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsar_b200.so")

SAR_OK = 0
SAR_NO_COMPENSATION = 1
SAR_OUTPUT_COMPLEX = 2
SAR_PROFILE_STAGES = 4
SAR_IMAGE_2D = 8
SAR_GRID_NUFFT = 16
SAR_REPORT_PEAK = 32
SAR_FORCE_PLAIN = 64
SAR_CUDA_GRAPH = 128
SAR_GRID_NEAREST = 256
SAR_STOLT_NUFFT = 512
STAGE_NAMES = ("K1 correct+x-FFT", "K2 y-FFT", "K3 filter+Stolt+z-IFFT", "K4a y-IFFT", "K4b x-IFFT+|.|")


class SarError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} [status {status}]")
        self.status = status


class GeomDesc(C.Structure):
    _fields_ = [("n_frames", C.c_int32), ("n_tx", C.c_int32), ("n_rx", C.c_int32),
                ("tx_xyz", C.POINTER(C.c_double)), ("rx_xyz", C.POINTER(C.c_double)),
                ("npx", C.c_int32), ("npy", C.c_int32),
                ("x0", C.c_double), ("y0", C.c_double), ("dx", C.c_double), ("dy", C.c_double),
                ("scan_xyz", C.POINTER(C.c_double)), ("z0", C.POINTER(C.c_double)),
                ("n_k", C.c_int32), ("k", C.POINTER(C.c_double)), ("pulse", C.POINTER(C.c_double)),
                ("device", C.c_int32)]


class ImageDesc(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("dz", C.c_double), ("z_ref", C.c_double), ("z_planes", C.POINTER(C.c_double))]


class PlanInfo(C.Structure):
    _fields_ = [("n_pairs", C.c_int32), ("jx_min", C.c_int32), ("jy_min", C.c_int32),
                ("nvx", C.c_int32), ("nvy", C.c_int32), ("roll_x", C.c_int32), ("roll_y", C.c_int32),
                ("axes", C.c_double * 6), ("k0", C.c_double), ("dk", C.c_double),
                ("workspace_bytes", C.c_size_t)]


class SlabDesc(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libsar_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_2305_02064_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    vp, i32, u32 = C.c_void_p, C.c_int32, C.c_uint32
    sig = {
        "sar_plan_describe": (C.c_int, [C.POINTER(GeomDesc), C.POINTER(ImageDesc), u32, C.POINTER(PlanInfo),
                                         vp, vp, vp, vp, vp, vp, vp]),
        "sar_plan_create": (C.c_int, [C.POINTER(vp), C.POINTER(GeomDesc), C.POINTER(ImageDesc), u32]),
        "sar_reconstruct": (C.c_int, [vp, vp, vp, vp]),
        "sar_reconstruct_host": (C.c_int, [vp, vp, vp, vp]),
        "sar_plan_describe_stolt_ranges": (C.c_int, [C.POINTER(GeomDesc), C.POINTER(ImageDesc), u32, vp]),
        "sar_plan_describe_nearest": (C.c_int, [C.POINTER(GeomDesc), C.POINTER(ImageDesc), u32, vp, vp]),
        "sar_plan_destroy": (C.c_int, [vp]),
        "sar_plan_get_axes": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "sar_plan_workspace_bytes": (C.c_int, [vp, C.POINTER(C.c_size_t)]),
        "sar_plan_profile_read": (C.c_int, [vp, C.POINTER(C.c_float), C.POINTER(i32)]),
        "sar_plan_profile_reset": (C.c_int, [vp]),
        "sar_plan_launches_per_call": (C.c_int, [vp, C.POINTER(i32)]),
        "sar_plan_peaks": (C.c_int, [vp, C.POINTER(C.c_float)]),
        "sar_debug_stage": (C.c_int, [vp, i32, vp, vp, vp]),
        "sar_debug_node_offsets": (C.c_int, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]),
        "sar_debug_stolt_index": (C.c_int, [vp, vp, i32, vp, vp, vp]),
        "sar_plan_create_slab": (C.c_int, [C.POINTER(vp), C.POINTER(GeomDesc), C.POINTER(ImageDesc), u32,
                                           C.POINTER(SlabDesc)]),
        "sar_slab_buffer_bytes": (C.c_int, [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
        "sar_slab_stage": (C.c_int, [vp, i32, vp, vp, vp, vp]),
        "sar_slab_stage_peers": (C.c_int, [vp, i32, vp, C.POINTER(vp), vp]),
        "sar_bpa": (C.c_int, [C.POINTER(GeomDesc), i32, vp, vp, C.c_int64, vp, vp, C.POINTER(C.c_float)]),
        "sar_status_string": (C.c_char_p, [C.c_int]),
        "sar_last_error": (C.c_char_p, []),
        "sar_version": (C.c_int, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    """Names of the C entry points this binding expects (the header's API)."""
    return ["sar_plan_describe", "sar_plan_describe_stolt_ranges", "sar_plan_describe_nearest", "sar_plan_create", "sar_reconstruct", "sar_reconstruct_host", "sar_plan_destroy",
            "sar_plan_get_axes", "sar_plan_workspace_bytes", "sar_plan_profile_read",
            "sar_plan_profile_reset", "sar_plan_launches_per_call", "sar_plan_peaks", "sar_debug_stage",
            "sar_debug_node_offsets", "sar_debug_stolt_index", "sar_plan_create_slab", "sar_slab_buffer_bytes",
            "sar_slab_stage", "sar_slab_stage_peers", "sar_bpa", "sar_status_string",
            "sar_last_error", "sar_version"]


def _check(status):
    if status != SAR_OK:
        lib = load_library()
        raise SarError(status, f"{lib.sar_status_string(status).decode()}: {lib.sar_last_error().decode()}")


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _descriptors(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref, pulse, device,
                 z_planes=None):
    keep = []

    def arr(a):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        keep.append(a)
        return a

    tx, rx, scan, k = arr(tx), arr(rx), arr(scan), arr(k)
    g = GeomDesc()
    g.n_frames = scan.shape[0] if scan.ndim == 3 else 0
    g.n_tx, g.n_rx = tx.shape[0], rx.shape[0]
    g.tx_xyz, g.rx_xyz = _dptr(tx), _dptr(rx)
    g.npx, g.npy = int(npx), int(npy)
    g.x0, g.y0, g.dx, g.dy = float(x0), float(y0), float(dx), float(dy)
    g.scan_xyz = _dptr(scan)
    g.z0 = _dptr(arr(z0)) if z0 is not None else None
    g.n_k = k.shape[0]
    g.k = _dptr(k)
    if pulse is not None:
        pc = np.asarray(pulse, dtype=np.complex128)
        g.pulse = _dptr(arr(np.stack([pc.real, pc.imag], axis=-1)))
    g.device = int(device)
    im = ImageDesc(int(nx), int(ny), int(nz), float(dz), float(z_ref))
    if z_planes is not None:
        zp = arr(np.atleast_1d(z_planes))
        im.nz = zp.shape[0]
        im.z_planes = _dptr(zp)
    return g, im, keep


def describe(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref, pulse=None, flags=0):
    """Host-only decomposition (``sar_plan_describe``): returns a dict with the
    integer node offsets, rolls, axes and the fp64 k tables -- no GPU needed."""
    lib = load_library()
    g, im, keep = _descriptors(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref, pulse, 0)
    npair = g.n_tx * g.n_rx
    jx, jy = np.zeros(npair, np.int32), np.zeros(npair, np.int32)
    kx, ky, kz = np.zeros(int(nx)), np.zeros(int(ny)), np.zeros(int(nz))
    F, P = g.n_frames, g.npx * g.npy
    ap, bp = np.zeros(max(F * P, 1), np.float32), np.zeros(max(F * npair, 1), np.float32)
    info = PlanInfo()
    vp = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
    _check(lib.sar_plan_describe(C.byref(g), C.byref(im), C.c_uint32(flags), C.byref(info), vp(jx), vp(jy),
                                 vp(kx), vp(ky), vp(kz), vp(ap), vp(bp)))
    del keep
    shp = (g.n_tx, g.n_rx)
    return dict(jx=jx.reshape(shp), jy=jy.reshape(shp), jx_min=info.jx_min, jy_min=info.jy_min,
                nvx=info.nvx, nvy=info.nvy, roll_x=info.roll_x, roll_y=info.roll_y, axes=tuple(info.axes),
                k0=info.k0, dk=info.dk, workspace_bytes=info.workspace_bytes, kx=kx, ky=ky, kz=kz,
                apose=ap[:F * P].reshape(F, P), bpair=bp[:F * npair].reshape(F, *shp))


def describe_stolt_ranges(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref, pulse=None,
                          flags=0):
    """Host-only (``sar_plan_describe_stolt_ranges``): int32 [ny, nx, 2] = the
    (jlo, jhi) k_z bin range step 3 evaluates for every spectral column,
    (0, -1) for a column the plan skips (zero Stolt output)."""
    lib = load_library()
    g, im, keep = _descriptors(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref, pulse, 0)
    out = np.zeros((int(ny), int(nx), 2), np.int32)
    _check(lib.sar_plan_describe_stolt_ranges(C.byref(g), C.byref(im), C.c_uint32(flags),
                                              C.c_void_p(out.ctypes.data)))
    del keep
    return out


def describe_nearest(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref, pulse=None, flags=0):
    """Host-only (``sar_plan_describe_nearest``): the SAR_GRID_NEAREST pose
    nodes (ix, iy), int32 [F, P] each (reading R20)."""
    lib = load_library()
    g, im, keep = _descriptors(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref, pulse, 0)
    F, P = g.n_frames, g.npx * g.npy
    ix, iy = np.zeros((max(F, 1), P), np.int32), np.zeros((max(F, 1), P), np.int32)
    _check(lib.sar_plan_describe_nearest(C.byref(g), C.byref(im), C.c_uint32(flags), C.c_void_p(ix.ctypes.data),
                                         C.c_void_p(iy.ctypes.data)))
    del keep
    return ix[:F], iy[:F]


def describe_nearest_scene(sc, flags=0):
    return describe_nearest(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, sc.x0, sc.y0, sc.dx, sc.dy, sc.z0, sc.k,
                            sc.nx, sc.ny, sc.nz, sc.dz_img, sc.z_ref, flags=flags)


def describe_scene(sc, flags=0):
    return describe(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, sc.x0, sc.y0, sc.dx, sc.dy, sc.z0, sc.k,
                    sc.nx, sc.ny, sc.nz, sc.dz_img, sc.z_ref, flags=flags)


def describe_stolt_ranges_scene(sc, flags=0):
    return describe_stolt_ranges(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, sc.x0, sc.y0, sc.dx, sc.dy, sc.z0, sc.k,
                                 sc.nx, sc.ny, sc.nz, sc.dz_img, sc.z_ref, flags=flags)


def bpa(tx, rx, scan, npx, npy, k, data, voxels, frame=0, out=None, stream=None, device=0):
    """Back-projection baseline (``sar_bpa``; the paper's comparison system,
    P:199-200): o(v) = sum s exp(+j k (|v-T| + |v-R|)) at the world positions
    ``voxels`` [V, 3] (host float64) from the device tensor ``data``
    [F, n_tx, n_rx, P, n_k] complex64.  Returns (complex64 [V] device tensor,
    kernel ms).  Synchronous."""
    import torch
    lib = load_library()
    k = np.asarray(k, dtype=np.float64)
    scan = np.asarray(scan, dtype=np.float64)
    g, _, keep = _descriptors(tx, rx, scan, npx, npy, 0.0, 0.0, 1.0, 1.0, None, k, 2, 2, 2, 1.0, 1.0, None, device)
    shape = (g.n_frames, g.n_tx, g.n_rx, g.npx * g.npy, g.n_k)
    if not (isinstance(data, torch.Tensor) and data.is_cuda and data.dtype == torch.complex64
            and tuple(data.shape) == shape and data.is_contiguous()):
        raise ValueError(f"data must be a contiguous CUDA complex64 tensor of shape {shape}")
    vox = np.ascontiguousarray(np.asarray(voxels, dtype=np.float64).reshape(-1, 3))
    n = vox.shape[0]
    if out is None:
        out = torch.empty(n, dtype=torch.complex64, device=data.device)
    elif not (out.is_cuda and out.dtype == torch.complex64 and out.numel() == n and out.is_contiguous()):
        raise ValueError("out must be a contiguous CUDA complex64 tensor with one element per voxel")
    ms = C.c_float(0.0)
    _check(lib.sar_bpa(C.byref(g), C.c_int32(frame), C.c_void_p(data.data_ptr()), C.c_void_p(vox.ctypes.data),
                       C.c_int64(n), C.c_void_p(out.data_ptr()), _stream_ptr(stream), C.byref(ms)))
    del keep
    return out, float(ms.value)


def bpa_scene(sc, data, voxels, frame=0, **kw):
    """``bpa`` for any object with the attributes of ``scenes.Scene``."""
    return bpa(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, sc.k, data, voxels, frame=frame, **kw)


class Plan:
    """A reconstruction plan (``sar_plan_create``).  Host arrays are copied by
    the library; the plan owns the device tables and workspace."""

    def __init__(self, tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref,
                 pulse=None, flags=0, device=0, z_planes=None, slab=None):
        """``z_planes`` (m) selects the 2-D single-plane mode (SAR_IMAGE_2D): the
        image is then [F, len(z_planes), ny, nx] and nz/dz are ignored.  ``slab``
        = (rank, world) creates one rank's plan of the single-image slab
        decomposition (``sar_plan_create_slab``; see ``SlabPlan``)."""
        lib = load_library()
        self._lib = lib
        if z_planes is not None:
            flags |= SAR_IMAGE_2D
        g, im, keep = _descriptors(tx, rx, scan, npx, npy, x0, y0, dx, dy, z0, k, nx, ny, nz, dz, z_ref,
                                   pulse, device, z_planes)
        h = C.c_void_p()
        if slab is None:
            _check(lib.sar_plan_create(C.byref(h), C.byref(g), C.byref(im), C.c_uint32(flags)))
        else:
            sd = SlabDesc(int(slab[0]), int(slab[1]))
            _check(lib.sar_plan_create_slab(C.byref(h), C.byref(g), C.byref(im), C.c_uint32(flags), C.byref(sd)))
        del keep
        self._h = h
        self.flags = flags
        self.device = device
        self.n_frames, self.n_tx, self.n_rx = g.n_frames, g.n_tx, g.n_rx
        self.npx, self.npy, self.n_k = g.npx, g.npy, g.n_k
        self.nx, self.ny, self.nz = im.nx, im.ny, im.nz

    @classmethod
    def from_scene(cls, sc, flags=0, device=0, pulse=None, z_planes=None, **kw):
        """Plan for any object with the attributes of ``scenes.Scene``."""
        return cls(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, sc.x0, sc.y0, sc.dx, sc.dy, sc.z0, sc.k,
                   sc.nx, sc.ny, sc.nz, sc.dz_img, sc.z_ref, pulse=pulse, flags=flags, device=device,
                   z_planes=z_planes, **kw)

    # ---- shapes -------------------------------------------------------------
    @property
    def data_shape(self):
        return (self.n_frames, self.n_tx, self.n_rx, self.npx * self.npy, self.n_k)

    @property
    def image_shape(self):
        return (self.n_frames, self.nz, self.ny, self.nx)

    def _check_tensor(self, t, shape, dtype, what):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{what} must be a CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"{what} is on cuda:{t.device.index}, plan on cuda:{self.device}")
        if tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous():
            raise ValueError(f"{what}: expected contiguous {dtype} {tuple(shape)}, got {t.dtype} {tuple(t.shape)}")

    # ---- execution ----------------------------------------------------------
    def reconstruct(self, data, out=None, stream=None):
        """Enqueue the reconstruction of device tensor ``data`` (complex64
        [F,n_tx,n_rx,P,n_k]) into ``out`` (float32 [F,nz,ny,nx], or complex64
        with SAR_OUTPUT_COMPLEX) on ``stream`` (default: torch's current)."""
        import torch
        self._check_tensor(data, self.data_shape, torch.complex64, "data")
        odt = torch.complex64 if self.flags & SAR_OUTPUT_COMPLEX else torch.float32
        if out is None:
            out = torch.empty(self.image_shape, dtype=odt, device=data.device)
        self._check_tensor(out, self.image_shape, odt, "out")
        _check(self._lib.sar_reconstruct(self._h, C.c_void_p(data.data_ptr()), C.c_void_p(out.data_ptr()),
                                         _stream_ptr(stream)))
        return out

    def reconstruct_host(self, data, out=None, stream=None):
        """End-to-end call with HOST buffers (numpy arrays or CPU tensors,
        pinned for full bandwidth); blocks until ``out`` is written."""
        import torch
        if isinstance(data, np.ndarray):
            data = torch.from_numpy(data)
        if data.is_cuda or tuple(data.shape) != self.data_shape or data.dtype != torch.complex64 \
                or not data.is_contiguous():
            raise ValueError("data must be a contiguous complex64 host array of shape %s" % (self.data_shape,))
        odt = torch.complex64 if self.flags & SAR_OUTPUT_COMPLEX else torch.float32
        if out is None:
            out = torch.empty(self.image_shape, dtype=odt)
        if isinstance(out, np.ndarray):
            out = torch.from_numpy(out)
        if out.is_cuda or tuple(out.shape) != self.image_shape or out.dtype != odt or not out.is_contiguous():
            raise ValueError("out must be a contiguous host array of shape %s" % (self.image_shape,))
        _check(self._lib.sar_reconstruct_host(self._h, C.c_void_p(data.data_ptr()), C.c_void_p(out.data_ptr()),
                                              _stream_ptr(stream)))
        return out

    # ---- queries ------------------------------------------------------------
    def axes(self):
        a = (C.c_double * 6)()
        _check(self._lib.sar_plan_get_axes(self._h, a))
        return tuple(a)

    def workspace_bytes(self):
        n = C.c_size_t()
        _check(self._lib.sar_plan_workspace_bytes(self._h, C.byref(n)))
        return n.value

    def launches_per_call(self):
        n = C.c_int32()
        _check(self._lib.sar_plan_launches_per_call(self._h, C.byref(n)))
        return n.value

    def peaks(self):
        """max |image| per frame of the last call (plans made with SAR_REPORT_PEAK)."""
        out = (C.c_float * max(self.n_frames, 1))()
        _check(self._lib.sar_plan_peaks(self._h, out))
        return np.array(out[:self.n_frames], dtype=np.float32)

    def profile_reset(self):
        _check(self._lib.sar_plan_profile_reset(self._h))

    def profile_read(self):
        ms = (C.c_float * 5)()
        n = C.c_int32()
        _check(self._lib.sar_plan_profile_read(self._h, ms, C.byref(n)))
        return list(ms), n.value

    # ---- debug / parity -----------------------------------------------------
    def debug_stage(self, stage, data, stream=None):
        import torch
        self._check_tensor(data, self.data_shape, torch.complex64, "data")
        F, ny, nx = self.n_frames, self.ny, self.nx
        shape = {1: (F, ny, nx, self.n_k), 2: (F, ny, nx, self.n_k), 3: (F, ny, nx, self.nz),
                 4: (F, self.nz, ny, nx)}[stage]
        out = torch.empty(shape, dtype=torch.complex64, device=data.device)
        _check(self._lib.sar_debug_stage(self._h, int(stage), C.c_void_p(data.data_ptr()),
                                         C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def node_offsets(self):
        n = self.n_tx * self.n_rx
        jx, jy = (C.c_int32 * n)(), (C.c_int32 * n)()
        mx, my = C.c_int32(), C.c_int32()
        _check(self._lib.sar_debug_node_offsets(self._h, jx, jy, C.byref(mx), C.byref(my)))
        shp = (self.n_tx, self.n_rx)
        return np.array(jx).reshape(shp), np.array(jy).reshape(shp), mx.value, my.value

    def stolt_index(self, cols, stream=None):
        """cols: int array [n, 2] of (a, b) spectral indices -> (i0 [n,nz], tau [n,nz])."""
        import torch
        cols = torch.as_tensor(np.ascontiguousarray(cols, dtype=np.int32)).to(f"cuda:{self.device}")
        n = cols.shape[0]
        i0 = torch.empty((n, self.nz), dtype=torch.int32, device=cols.device)
        tau = torch.empty((n, self.nz), dtype=torch.float32, device=cols.device)
        _check(self._lib.sar_debug_stolt_index(self._h, C.c_void_p(cols.data_ptr()), int(n),
                                               C.c_void_p(i0.data_ptr()), C.c_void_p(tau.data_ptr()),
                                               _stream_ptr(stream)))
        return i0, tau

    def close(self):
        if getattr(self, "_h", None):
            _check(self._lib.sar_plan_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class SlabPlan(Plan):
    """One rank of the single-image slab decomposition (``sar_plan_create_slab``,
    SURVEY 8(e)): stage 1 (K1 on this rank's lattice rows, packed per
    destination), exchange #1, stage 2 (y-FFT, filter + Stolt + z-IFFT, y-IFFT
    on this rank's k_x columns, packed), exchange #2, stage 3 (x-IFFT +
    magnitude of this rank's z-slots into the image).  The exchanges are the
    caller's (``paper_2305_02064_b200.slab``)."""

    def __init__(self, *args, rank=0, world=1, **kw):
        super().__init__(*args, slab=(rank, world), **kw)
        self.rank, self.world = rank, world
        G = world
        self.send1_shape = (G, self.ny // G, self.nx // G, self.n_k)
        self.send2_shape = (G, self.ny, self.nx // G, self.nz // G)
        b1, b2 = C.c_size_t(), C.c_size_t()
        _check(self._lib.sar_slab_buffer_bytes(self._h, C.byref(b1), C.byref(b2)))
        assert b1.value == 8 * int(np.prod(self.send1_shape)) and b2.value == 8 * int(np.prod(self.send2_shape))

    @classmethod
    def from_scene(cls, sc, rank=0, world=1, flags=0, device=0, pulse=None):
        return cls(sc.tx, sc.rx, sc.scan, sc.npx, sc.npy, sc.x0, sc.y0, sc.dx, sc.dy, sc.z0, sc.k,
                   sc.nx, sc.ny, sc.nz, sc.dz_img, sc.z_ref, pulse=pulse, flags=flags, device=device,
                   rank=rank, world=world)

    def _stage(self, stage, a, b, img, stream):
        _check(self._lib.sar_slab_stage(self._h, stage, C.c_void_p(a.data_ptr()),
                                        C.c_void_p(b.data_ptr() if b is not None else 0),
                                        C.c_void_p(img.data_ptr() if img is not None else 0), _stream_ptr(stream)))

    def stage1(self, data, out=None, stream=None):
        import torch
        self._check_tensor(data, self.data_shape, torch.complex64, "data")
        if out is None:
            out = torch.empty(self.send1_shape, dtype=torch.complex64, device=data.device)
        self._check_tensor(out, self.send1_shape, torch.complex64, "out")
        self._stage(1, data, out, None, stream)
        return out

    def stage2(self, recv1, out=None, stream=None):
        """``recv1`` (exchange #1 result, [G, ny/G, nx/G, n_k]) is overwritten."""
        import torch
        self._check_tensor(recv1, self.send1_shape, torch.complex64, "recv1")
        if out is None:
            out = torch.empty(self.send2_shape, dtype=torch.complex64, device=recv1.device)
        self._check_tensor(out, self.send2_shape, torch.complex64, "out")
        self._stage(2, recv1, out, None, stream)
        return out

    def stage3(self, recv2, image, stream=None):
        """Writes this rank's nz/G planes of ``image`` ([1, nz, ny, nx])."""
        import torch
        self._check_tensor(recv2, self.send2_shape, torch.complex64, "recv2")
        odt = torch.complex64 if self.flags & SAR_OUTPUT_COMPLEX else torch.float32
        self._check_tensor(image, self.image_shape, odt, "image")
        self._stage(3, recv2, None, image, stream)
        return image

    def stage_peers(self, stage, inp, peer_ptrs, stream=None):
        """Stage 1 (inp = data) or 2 (inp = this rank's exchange-#1 receive
        buffer, overwritten) with the exchange done by stores: block h goes
        straight into slot ``rank`` of ``peer_ptrs[h]`` (device addresses of
        every rank's receive buffer, valid in this process)."""
        import torch
        if stage == 1:
            self._check_tensor(inp, self.data_shape, torch.complex64, "data")
        else:
            self._check_tensor(inp, self.send1_shape, torch.complex64, "recv1")
        if len(peer_ptrs) != self.world:
            raise ValueError("need one receive buffer per rank")
        arr = (C.c_void_p * self.world)(*[C.c_void_p(int(x)) for x in peer_ptrs])
        _check(self._lib.sar_slab_stage_peers(self._h, stage, C.c_void_p(inp.data_ptr()), arr,
                                              _stream_ptr(stream)))

    def planes(self):
        """Output planes this rank writes: (z + nz/2) mod nz of its z-slots (reading R8)."""
        nzl = self.nz // self.world
        return [(z + self.nz // 2) % self.nz for z in range(self.rank * nzl, (self.rank + 1) * nzl)]
