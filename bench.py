#!/usr/bin/env python
"""Benchmark of the B200 reconstruction path (BASELINE.json metric:
"ms per 3-D image; Gsamples/s; achieved HBM GB/s vs B200 peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config large]
    python bench.py --impl reference ...      # the fp64 CPU oracle arm

A step is one sar_reconstruct call over the whole workload (all 5 kernels:
correction+x-FFT, y-FFT, filter+Stolt+z-IFFT, y-IFFT, x-IFFT+magnitude) with
the input already resident in HBM.  The default workload is Large
(BASELINE.json configs[3], the config the north-star roofline target is
quoted on; 12 GiB of raw samples, larger than the 126 MB L2, so no flush is
needed between steps).  Under torchrun every rank reconstructs its own replica
(the path is one GPU per image: "replicas only") and rank 0
prints one JSON line with the max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import dataclasses  # noqa: E402

import numpy as np  # noqa: E402

METRIC = "Gsamples/s (raw complex64 samples reconstructed into 3-D images per second)"
UNIT = "Gsamples/s"
FALLBACK_HBM_GBS = 6650.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def stage_alg_bytes(sc):
    """Algorithmic bytes per launch of each kernel slot:
    the compulsory read of its input and write of its output, 8 B per complex64
    element, 4 B per float32 voxel."""
    F, ny, nx, nk, nz = sc.n_frames, sc.ny, sc.nx, sc.n_k, sc.nz
    planar = 8 * F * ny * nx * nk
    vol = 8 * F * ny * nx * nz
    img = 4 * F * nz * ny * nx
    return [sc.raw_bytes() + planar, 2 * planar, planar + vol, 2 * vol, vol + img]


def stage_slots(plan, sar):
    """(slot index, name) of the kernel slots one call times."""
    return list(enumerate(sar.STAGE_NAMES))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_info():
    """CPU model, logical cores and RAM of this host (for the cpu_baseline line)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        import psutil
        ram = round(psutil.virtual_memory().total / 2**30, 1)
    except ImportError:
        pass
    return {"cpu_model": model, "cores": os.cpu_count(), "ram_GiB": ram}


def oracle_sample(sc, s_host, planes=None, nufft=False, nearest=False, stolt_nufft=False):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload:
    Tx/Rx channel (0,0) through the whole path.  The oracle's per-channel
    work (O1-O2 compensation + lattice accumulation; the NUFFT spread) and
    its once-per-image work (FT_2D, filter, Stolt, IFT_3D, magnitude) are
    timed separately, so the full image's oracle time is projected as
    n_channels * t_channel + t_image.  ``sc`` is the 3-D scene, ``s_host``
    its channel (0,0).  Returns a dict of the times (s) and the projection."""
    import oracle
    geo = oracle.decompose(sc.tx[:1], sc.rx[:1], sc.scan, sc.npx, sc.npy, sc.x0, sc.y0, sc.dx, sc.dy,
                           sc.z0, sc.k, sc.nx, sc.ny, sc.nz, sc.dz_img, sc.z_ref)
    sc1 = dataclasses.replace(sc, tx=sc.tx[:1], rx=sc.rx[:1])
    t0 = time.perf_counter()
    if nufft:
        S, g1 = oracle.nufft.spectrum_nufft(s_host, sc1)
        t1 = time.perf_counter()
        Fk = oracle.rma_filter(S, g1)
        if planes:
            oracle.magnitude_planes(oracle.ifft2_planes(oracle.plane_sum(Fk, g1, planes)), g1)
        else:
            oracle.magnitude_image(oracle.ifft3(oracle.stolt(Fk, g1)), g1)
    else:
        nodes = oracle.nearest_nodes(sc.scan, sc.x0, sc.y0, sc.dx, sc.dy) if nearest else None
        planar = oracle.compensate(s_host, geo, nodes=nodes)
        t1 = time.perf_counter()
        Fk = oracle.rma_filter(oracle.fft2(planar), geo)
        if planes:
            oracle.magnitude_planes(oracle.ifft2_planes(oracle.plane_sum(Fk, geo, planes)), geo)
        elif stolt_nufft:
            import scipy.fft
            oz = oracle.stolt_nufft.stolt_nufft(Fk, geo)
            oracle.magnitude_image(scipy.fft.ifft2(oz, axes=(1, 2), workers=os.cpu_count()), geo)
        else:
            oracle.magnitude_image(oracle.ifft3(oracle.stolt(Fk, geo)), geo)
    t2 = time.perf_counter()
    nch = sc.n_tx * sc.n_rx
    return {"t_channel": t1 - t0, "t_image": t2 - t1, "t_sample": t2 - t0, "n_channels": nch,
            "t_projected": nch * (t1 - t0) + (t2 - t1), "samples_sample": int(np.prod(s_host.shape)),
            "samples_image": sc.n_samples}


def oracle_line(sc, name, res, planes=None, nufft=False):
    """cpu_baseline object for an oracle_sample result."""
    what = ("NUFFT spectrum + " if nufft else "O1-O2 + ") + \
        (f"O3-O4, O5'-O7' on {len(planes)} plane(s)" if planes else
         f"O3-O7 incl. the {sc.nx}x{sc.ny}x{sc.nz} RMA")
    return dict(value=res["samples_image"] / res["t_projected"] / 1e9, unit=UNIT, kind="oracle",
                **host_info(),
                sample=(f"{name}: fp64 oracle ({what}) timed on Tx/Rx channel (0,0) "
                        f"({res['samples_sample']} of {res['samples_image']} samples): per-channel part "
                        f"{res['t_channel']:.3g} s, once-per-image part {res['t_image']:.3g} s; the full image "
                        f"projected as {res['n_channels']} x {res['t_channel']:.3g} + {res['t_image']:.3g} = "
                        f"{res['t_projected']:.3g} s (value = image samples / projected time)"),
                seconds_measured=res["t_sample"], seconds_projected_full_image=res["t_projected"])


def run_reference(args):
    """--impl reference: the oracle arm (fp64 CPU), rank 0 only."""
    rank, world, _ = _dist()
    if rank != 0:
        return
    import scenes
    sc = scenes.make_scene(args.config)
    # a one-channel sample needs only that channel's echo: synthesise it on the
    # CPU when feasible, else on the GPU
    sub = dataclasses.replace(sc, tx=sc.tx[:1], rx=sc.rx[:1])
    if sub.n_samples * max(len(q) for q in sub.scat_pos) <= 5e8:
        s = scenes.synthesize_cpu(sub)
    else:
        import scenes.gpu
        scenes.gpu.build()
        s = scenes.gpu.synthesize_gpu(sub).cpu().numpy()
    for _ in range(args.warmup):
        oracle_sample(sc, s)
    res = None
    tproj = []
    for _ in range(args.steps):
        res = oracle_sample(sc, s)
        tproj.append(res["t_projected"])
    t = float(np.sum(tproj))
    val = sc.n_samples * args.steps / t / 1e9
    cpu = oracle_line(sc, args.config, res)
    sample = cpu["sample"]
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "sample": sample},
            "cpu_baseline": dict(cpu, value=val),
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import scenes
    import scenes.gpu
    import paper_2305_02064_b200 as sar
    from paper_2305_02064_b200 import build as sbuild

    rank, world, local = _dist()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        sbuild.build()
        scenes.gpu.build()
    if world > 1:
        dist.barrier()

    full = scenes.make_scene(args.config)
    # a batch of independent frames is split across ranks (no collective on the
    # data path, "strong" scaling); a single image is replicated ("weak")
    from paper_2305_02064_b200.shard import frame_range, max_over_ranks
    sharded = world > 1 and full.n_frames > 1
    if sharded:
        lo, hi = frame_range(full.n_frames, rank, world)
        sc = scenes.frame_subset(full, lo, hi)
    else:
        sc = full
    data = scenes.gpu.synthesize_gpu(sc, device=local)
    planes = [float(z) for z in args.planes.split(",")] if args.planes else None
    sc3 = sc
    if planes:
        sc = dataclasses.replace(sc, nz=len(planes))       # image [F][planes][ny][nx]
    gflag = {"nufft": sar.SAR_GRID_NUFFT, "nearest": sar.SAR_GRID_NEAREST}.get(args.grid, 0)
    if args.stolt == "nufft":
        gflag |= sar.SAR_STOLT_NUFFT
    # the timed plan records no per-kernel events (they would sit between the
    # programmatically dependent launches); a second, profiled plan measures
    # the per-kernel times after the timed region
    plan = sar.Plan.from_scene(sc, flags=gflag, device=local, z_planes=planes)
    out = torch.empty(sc.image_shape, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        plan.reconstruct(data, out, stream)
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            plan.reconstruct(data, out, stream)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    with sar.Plan.from_scene(sc, flags=sar.SAR_PROFILE_STAGES | gflag, device=local, z_planes=planes) as pplan:
        for _ in range(2):
            pplan.reconstruct(data, out, stream)
        torch.cuda.synchronize(dev)
        pplan.profile_reset()
        for _ in range(max(3, min(args.steps, 10))):
            pplan.reconstruct(data, out, stream)
        stage_ms, ncalls = pplan.profile_read()
    ms_total = max_over_ranks(ms_total, dist if world > 1 else None, dev)
    ms_step = ms_total / args.steps
    samples = full.n_samples if sharded else sc.n_samples * world   # all ranks
    value = samples / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel (largest share of the step)
    peak, peak_src = _peaks()
    slots = stage_slots(plan, sar)
    avg = [m / max(ncalls, 1) for m in stage_ms]
    tot = sum(avg[i] for i, _ in slots)
    dom, dom_name = max(slots, key=lambda x: avg[x[0]])
    alg = stage_alg_bytes(sc)
    ach = alg[dom] / (avg[dom] * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"{args.config}_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(str(dom))
    path_gbs = sc.alg_bytes() / (ms_step * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": dom_name, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "traffic": traffic, "alg_bytes": alg[dom], "ms": avg[dom], "peak_source": peak_src}
    if dom == 0:
        # K1: SURVEY 8(d) counts the raw samples it reads as algorithmic; the W0
        # volume it writes is an intermediate (an implementation choice), kept
        # as a second figure (round-1 verdict)
        raw = sc.raw_bytes()
        roof.update({"achieved": raw / (avg[dom] * 1e-3) / 1e9, "frac": raw / (avg[dom] * 1e-3) / 1e9 / peak,
                     "alg_bytes": raw, "achieved_incl_intermediate_write": ach,
                     "frac_incl_intermediate_write": ach / peak})
    if args.grid == "nufft" and dom == 0:
        # NUFFT spread (K1s) is FP32-FMA bound, not HBM bound: algorithmic
        # flops = samples x (2W+1)^2 taps x 4 (complex sample x real weight =
        # 2 FMA), W = 6; peak = 148 SMs x 128 FP32 lanes x 2 flop x the max SM
        # clock
        flops = sc.n_samples * 13 * 13 * 4
        fpeak = 148 * 128 * 2 * 1.965e9 / 1e12
        fach = flops / (avg[dom] * 1e-3) / 1e12
        roof = {"bound": "alu", "kernel": "K1s NUFFT spread (FP32 FMA)", "achieved": fach, "peak": fpeak,
                "unit": "TFLOP/s", "frac": fach / fpeak, "traffic": None, "alg_flops": flops, "ms": avg[dom],
                "peak_source": "derived: 148 SMs x 128 FP32 FMA/clk x 2 x 1.965 GHz"}
    ncu_bytes = None
    if traffic is not None:
        tj = json.load(open(tp))
        ncu_bytes = sum(int(tj[str(i)]) for i, _ in slots if str(i) in tj)

    # end-to-end through the public API with host buffers (pinned)
    e2e = None
    e2e_ok = not args.no_e2e
    if e2e_ok:
        # every rank of the node pins its inputs + image: skip (rather than
        # crash the node) when the host cannot hold them all
        try:
            import psutil
            need = world * (sc.raw_bytes() + sc.image_bytes())
            if psutil.virtual_memory().available < 1.3 * need:
                e2e_ok = False
                e2e = {"skipped": f"host RAM: {world} ranks x {(sc.raw_bytes() + sc.image_bytes()) / 2**30:.1f} GiB "
                                  f"pinned > available"}
        except ImportError:
            pass
    if e2e_ok:
        h_in = torch.empty(sc.data_shape, dtype=torch.complex64, pin_memory=True)
        h_in.copy_(data)
        h_out = torch.empty(sc.image_shape, dtype=torch.float32, pin_memory=True)
        plan2 = sar.Plan.from_scene(sc, flags=gflag, device=local, z_planes=planes)
        plan2.reconstruct_host(h_in, h_out, stream)  # warm-up (allocates staging)
        ke = max(1, min(args.steps, args.e2e_steps))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            plan2.reconstruct_host(h_in, h_out, stream)
        dt = (time.perf_counter() - t0) / ke
        if world > 1:
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": samples / dt / 1e9, "unit": UNIT, "ms_per_step": dt * 1e3,
               "h2d_bytes_per_step": sc.raw_bytes(), "d2h_bytes_per_step": sc.image_bytes(), "steps": ke}
        plan2.close()
        del h_in, h_out

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s_host = data[:, :1, :1].cpu().numpy()
        res = oracle_sample(sc3, s_host, planes=planes, nufft=args.grid == "nufft", nearest=args.grid == "nearest",
                            stolt_nufft=args.stolt == "nufft")
        cpu = oracle_line(sc3, args.config, res, planes=planes, nufft=args.grid == "nufft")

    # parity of this configuration as last measured by the GPU parity suite
    # (the full fp64 oracle on the host takes minutes: tests, not the bench)
    parity = None
    pp = os.path.join(ROOT, "profiles", f"{args.config}_parity.json")
    if os.path.exists(pp) and not planes and not gflag:
        parity = json.load(open(pp))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded scenes, GPU-synthesised Eq. (9) echo)",
            "config": {"workload": args.config + (f" 2-D planes {planes}" if planes else "") +
                       {"nufft": " NUFFT placement", "nearest": " NEAREST placement"}.get(args.grid, "") +
                       (" NUFFT Stolt" if args.stolt == "nufft" else ""),
                       "frames": sc.n_frames, "tx": sc.n_tx, "rx": sc.n_rx,
                       "poses": sc.n_pos, "n_k": sc.n_k, "image": [sc.nx, sc.ny, sc.nz],
                       "samples_per_step": samples, "raw_GiB_per_gpu": sc.raw_bytes() / 2**30,
                       "l2": "inputs larger than L2 (no flush)" if sc.raw_bytes() > 126e6 else "L2 not flushed",
                       "parallelism": (f"frames sharded x{world}" if sharded else f"replicas x{world}")},
            "ms_per_image": ms_step / (full.n_frames if sharded else sc.n_frames),
            "path": {"alg_bytes": sc.alg_bytes(), "achieved_GBps": path_gbs, "peak_GBps": peak,
                     "frac": path_gbs / peak, "frac_vs_spec_8TBps": path_gbs / 8000.0,
                     "ncu_dram_bytes": ncu_bytes,
                     "ncu_dram_GBps": (ncu_bytes / (ms_step * 1e-3) / 1e9) if ncu_bytes else None},
            "roofline": roof,
            "stages": {n: {"ms": avg[i], "share": avg[i] / max(tot, 1e-12),
                           "alg_GBps": alg[i] / (max(avg[i], 1e-9) * 1e-3) / 1e9} for i, n in slots},
            "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
            "gpu_launches": plan.launches_per_call() * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


# FP32 peak the ALU-bound lines report against:
# 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def run_bpa(args):
    """The GPU back-projection baseline (sar_bpa): a
    step is one call over --bpa-voxels image voxels (default: a z-centred slab of
    the config's image grid, at most 65536 voxels) against every sample of
    frame 0.  Single GPU (a baseline, not the product path)."""
    import torch
    import scenes
    import scenes.gpu
    import paper_2305_02064_b200 as sar
    from paper_2305_02064_b200 import build as sbuild

    rank, world, local = _dist()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    sbuild.build()
    scenes.gpu.build()
    sc = scenes.make_scene(args.config)
    d = scenes.gpu.synthesize_gpu(sc)
    with sar.Plan.from_scene(sc) as plan:
        x0, y0, z0, dx, dy, dz = plan.axes()
    nvox = args.bpa_voxels or min(sc.nx * sc.ny * sc.nz, 65536)
    planes = max(1, min(sc.nz, nvox // (sc.nx * sc.ny)))
    m0 = sc.nz // 2 - planes // 2
    m, iy, ix = np.meshgrid(np.arange(m0, m0 + planes), np.arange(sc.ny), np.arange(sc.nx), indexing="ij")
    vox = np.stack([x0 + ix * dx, y0 + iy * dy, z0 + m * dz], axis=-1).reshape(-1, 3)[:max(nvox, 1)]
    nvox = vox.shape[0]
    terms = nvox * sc.n_tx * sc.n_rx * sc.n_pos * sc.n_k
    out = torch.empty(nvox, dtype=torch.complex64, device=d.device)
    for _ in range(args.warmup):
        sar.bpa_scene(sc, d, vox, out=out)
    torch.cuda.synchronize()
    kms = []
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            kms.append(sar.bpa_scene(sc, d, vox, out=out)[1])
        e1.record()
        torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / args.steps
    kern = float(np.mean(kms))
    # e2e: host samples of the frame and host voxels in, host values out
    h = d[:1].cpu().pin_memory()
    sc1 = scenes.frame_subset(sc, 0, 1) if sc.n_frames > 1 else sc
    t0 = time.perf_counter()
    dd = h.to(d.device, non_blocking=True)
    res = sar.bpa_scene(sc1, dd, vox)[0].cpu()
    e2e_ms = (time.perf_counter() - t0) * 1e3
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        txw, rxw = scenes.element_positions(sc, 0)
        s0 = d[0].cpu().numpy()
        nv = max(1, min(nvox, int(2e9 // (terms // nvox))))   # ~2e9 terms: some 10-30 s of NumPy
        t0 = time.perf_counter()
        want = oracle.bpa(s0, txw, rxw, sc.k, vox[:nv])
        dt = time.perf_counter() - t0
        got = res[:nv].numpy().astype(np.complex128)
        cpu = {"value": nv * (terms // nvox) / dt / 1e9, "unit": "Gterms/s", "kind": "oracle",
               "sample": f"oracle.bpa on the first {nv} of the {nvox} voxels ({dt:.1f} s)",
               "rel_l2_of_gpu_vs_oracle_on_sample": float(np.linalg.norm(got - want) / np.linalg.norm(want)),
               **host_info()}
    flops = 8.0 * terms   # one complex multiply-add per term
    line = {
        "metric": "Gterms/s (back-projection terms s*exp(jkR) accumulated per second; BPA baseline)",
        "value": terms / (ms_step * 1e-3) / 1e9, "unit": "Gterms/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (k loop), f64 (distances, phase reduction, totals)",
        "data": "synthetic (seeded scenes, GPU-synthesised Eq. (9) echo)",
        "config": {"workload": f"{args.config} BPA baseline, {nvox} voxels ({planes} central z planes)",
                   "tx": sc.n_tx, "rx": sc.n_rx, "poses": sc.n_pos, "n_k": sc.n_k, "terms_per_step": terms,
                   "l2": "samples re-read by every CTA from L2 (ALU bound)"},
        "roofline": {"bound": "alu", "kernel": "k_bpa", "achieved": flops / (kern * 1e-3) / 1e12,
                     "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": flops / (kern * 1e-3) / 1e12 / FP32_PEAK_TFLOPS, "traffic": None, "ms": kern,
                     "alg_flops": flops, "peak_source": "148 SMs x 128 lanes x 2 x 1.965 GHz (DESIGN.md section 8)"},
        "full_image_projection_s": (sc.nx * sc.ny * sc.nz / nvox) * kern * 1e-3,
        "cpu_baseline": cpu,
        "e2e": {"value": terms / (e2e_ms * 1e-3) / 1e9, "unit": "Gterms/s", "ms": e2e_ms,
                "h2d_bytes_per_step": h.numel() * 8 + vox.nbytes, "d2h_bytes_per_step": nvox * 8},
        "gpu_launches": args.steps, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_slab(args):
    """One image split over the N ranks (single-image slab decomposition,
    sar_slab_stage + two NCCL all-to-alls): strong scaling of the Large
    image.  Every rank holds the raw samples of the image (K1 reads only the
    pose rows of its lattice rows)."""
    import torch
    import scenes
    import scenes.gpu
    import paper_2305_02064_b200 as sar
    from paper_2305_02064_b200 import build as sbuild, slab
    from paper_2305_02064_b200.shard import max_over_ranks

    rank, world, local = _dist()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        sbuild.build()
        scenes.gpu.build()
    if world > 1:
        dist.barrier()
    sc = scenes.make_scene(args.config)
    if sc.n_frames != 1:
        raise SystemExit("--slab splits one image: use a single-frame config")
    data = scenes.gpu.synthesize_gpu(sc, device=local)
    plan = sar.SlabPlan.from_scene(sc, rank=rank, world=world, device=local)
    image = torch.empty(sc.image_shape, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    xfn = slab.exchange if world > 1 else (lambda t, group=None: t)
    if args.p2p:
        # exchange by peer stores: the pack kernels write straight into every
        # rank's receive buffer (CUDA IPC over NVLink / NVSwitch)
        recv1 = torch.empty(plan.send1_shape, dtype=torch.complex64, device=dev)
        recv2 = torch.empty(plan.send2_shape, dtype=torch.complex64, device=dev)
        if world > 1:
            peers1, keep1 = slab.open_peer_buffers(recv1)
            peers2, keep2 = slab.open_peer_buffers(recv2)
        else:
            peers1, peers2 = [recv1.data_ptr()], [recv2.data_ptr()]

    def step():
        if not args.p2p:
            slab.reconstruct(plan, data, image, exchange_fn=xfn)
        elif world > 1:
            slab.reconstruct_peers(plan, data, image, recv1, recv2, peers1, peers2)
        else:
            plan.stage_peers(1, data, peers1)
            plan.stage_peers(2, recv1, peers2)
            plan.stage3(recv2, image)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    ms_total = max_over_ranks(ev0.elapsed_time(ev1), dist if world > 1 else None, dev)
    ms_step = ms_total / args.steps
    value = sc.n_samples / (ms_step * 1e-3) / 1e9
    peak, peak_src = _peaks()
    # per-rank algorithmic bytes: its share of the raw samples and of the image
    alg_rank = sc.alg_bytes() / world
    ach = alg_rank / (ms_step * 1e-3) / 1e9
    xbytes = 8 * (int(np.prod(plan.send1_shape)) + int(np.prod(plan.send2_shape)))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded scenes, GPU-synthesised Eq. (9) echo)",
            "config": {"workload": args.config + " single image split over the ranks",
                       "frames": 1, "tx": sc.n_tx, "rx": sc.n_rx, "poses": sc.n_pos, "n_k": sc.n_k,
                       "image": [sc.nx, sc.ny, sc.nz], "samples_per_step": sc.n_samples,
                       "l2": "inputs larger than L2 (no flush)",
                       "parallelism": f"slab x{world}: y-rows -> " + ("peer stores" if args.p2p else "all-to-all") +
                                      " -> k_x columns -> " + ("peer stores" if args.p2p else "all-to-all") + " -> z-slots",
                       "exchange_bytes_per_rank": xbytes},
            "ms_per_image": ms_step,
            "roofline": {"bound": "hbm", "kernel": "whole slab step (per rank)", "achieved": ach, "peak": peak,
                         "unit": "GB/s", "frac": ach / peak, "traffic": None, "alg_bytes": alg_rank,
                         "ms": ms_step, "peak_source": peak_src},
            "cpu_baseline": None, "e2e": None,
            "gpu_launches": 5 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="large", choices=["tiny", "small", "freehand", "large", "realtime"])
    ap.add_argument("--grid", default="raster", choices=["raster", "nufft", "nearest"],
                    help="in-plane placement: RASTER lattice (reading R7), FGG-NUFFT from the true positions (R19) "
                         "or the lattice node nearest the true position (NEAREST, R20)")
    ap.add_argument("--stolt", default="linear", choices=["linear", "nufft"],
                    help="Stolt step: linear pull onto the uniform k_z grid (reading R4) or the 1-D NUFFT from "
                         "the non-uniform k_z (SAR_STOLT_NUFFT, reading R21)")
    ap.add_argument("--planes", type=str, default=None,
                    help="comma-separated z planes (m): 2-D single-plane images (SAR_IMAGE_2D, Table I '2-D' rows) "
                         "instead of the 3-D volume")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--slab", action="store_true",
                    help="split ONE image over the ranks (slab decomposition, two all-to-alls; strong scaling)")
    ap.add_argument("--p2p", action="store_true",
                    help="with --slab: exchange by peer stores into IPC-mapped receive buffers instead of NCCL")
    ap.add_argument("--bpa", action="store_true",
                    help="time the GPU back-projection baseline (sar_bpa; the paper's comparison system, P:199-200) "
                         "instead of the reconstruction path")
    ap.add_argument("--bpa-voxels", type=int, default=0, help="with --bpa: voxels per step (default <= 65536)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 is below the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.bpa:
        run_bpa(args)
    elif args.slab:
        run_slab(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
