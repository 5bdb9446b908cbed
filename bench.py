#!/usr/bin/env python
"""bench.py -- TCo639 spherical-harmonics inverse+direct transform pair on N B200.

Metric (BASELINE.json): "TCo639 inverse+direct transform ms at 1/2/4/8 B200;
% FP64/HBM/NVLink roofline".  One step = one inv_trans + dir_trans pair over
NFLD = 548 synthetic fields (fixed across GPU counts, so
scaling is strong).  ``value`` = device time per pair (CUDA events around K
back-to-back pairs on the launching stream, max over ranks); inputs (1.8 GB
spectral, 7.3 GB grid) are far larger than the 126 MB L2, so no flush is
needed between steps.  ``e2e`` = the same pair through the public API with
the spectral input coming from pinned host memory and the spectral result
going back to it every step.

  python bench.py [--gpus N --steps K --warmup W]            our B200 path
  python bench.py --impl reference [...]                     CPU oracle arm

Under torchrun (N > 1) every rank drives one GPU through NCCL.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TCo639 inverse+direct transform ms at 1/2/4/8 B200; % FP64/HBM/NVLink roofline"
UNIT = "ms/pair"
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def parse():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--truncation", type=int, default=639)
    ap.add_argument("--nfld", type=int, default=548)
    ap.add_argument("--cpu-fields", type=int, default=137,
                    help="fields in the bounded CPU sample (137 = one model level set of the 548-field batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gp-layout", default=None,
                    help="nA,nB: grid side in the 2-D grid-point layout (adds the ring <-> grid-point transposition)")
    ap.add_argument("--recompute-legendre", action="store_true",
                    help="regenerate the P table chunk by chunk every transform (TCo1999 memory mode)")
    return ap.parse_args()


DEBUG_VARS = ("SHT_FFT_DEBUG", "SHT_LEG_DEBUG")


def refuse_debug() -> None:
    """Profiling switches that skip work inside the product kernels void a bench number."""
    bad = [v for v in DEBUG_VARS if os.environ.get(v, "0") not in ("", "0")]
    if bad:
        raise SystemExit(f"bench.py refuses to run with {', '.join(bad)} set (they skip work inside the kernels)")


def lscpu() -> dict:
    out = {"os_cpu_count": os.cpu_count()}
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in txt.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)",
                             "NUMA node(s)", "CPU max MHz"):
                out[k.strip()] = v.strip()
    except Exception:
        pass
    return out


def window_average(samples, t0: float, t1: float) -> float:
    """Mean power over [t0, t1], each sample held until the next one and the first one extended
    backwards -- a restatement of the reference's haloflow.energy.window_average
    (/root/reference/pkg/src/haloflow/energy.py:83-111); tests/test_bench.py checks it against the
    reference's own function."""
    if t1 <= t0 or not samples:
        raise ValueError("empty window or no samples")
    times = [t for t, _ in samples]
    if any(b <= a for a, b in zip(times, times[1:])):
        raise ValueError("samples must be in strictly increasing time order")
    import bisect

    joules, cursor = 0.0, t0
    while cursor < t1:
        i = max(bisect.bisect_right(times, cursor) - 1, 0)
        seg_end = times[i + 1] if i + 1 < len(times) else t1
        seg_end = min(max(seg_end, cursor), t1)
        if seg_end == cursor:
            seg_end = t1
        joules += samples[i][1] * (seg_end - cursor)
        cursor = seg_end
    return joules / (t1 - t0)


def peaks() -> dict:
    """Roofline denominators: measured HBM copy (MEASURED_PEAKS.json), measured
    DMMA issue peak (profiles/r01_probe_fp64.json), measured NVLink peer copy."""
    hbm, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    mp = ROOT / "MEASURED_PEAKS.json"
    if mp.exists():
        try:
            hbm, hbm_src = float(json.loads(mp.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
        except Exception:
            pass
    fp64, fp64_src = 37.14, "profiles/r01_probe_fp64.json (DMMA.8x8x4 issue peak, 1965 MHz)"
    pf = ROOT / "profiles" / "r01_probe_fp64.json"
    if pf.exists():
        try:
            d = json.loads(pf.read_text())
            fp64 = max(v for k, v in d.items() if k.startswith("dmma_") and isinstance(v, (int, float)))
        except Exception:
            pass
    return {"fp64_tflops": fp64, "fp64_src": fp64_src, "hbm_gbs": hbm, "hbm_src": hbm_src,
            "nvlink_gbs": NVLINK_GBS, "nvlink_src": "B200_PROFILING.md measured peer copy per direction"}


class Clocks:
    """nvidia-smi sampler of one GPU running during the timed region (every rank samples its own)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(gpu_index)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.t0 = self.t1 = None
        # NVML start-up must be over before the timed region: wait for the first samples
        t0 = time.perf_counter()
        while self.p is not None and time.perf_counter() - t0 < 5.0:
            if Path(self.f.name).stat().st_size > 0:
                break
            time.sleep(0.01)

    def mark(self) -> None:
        """Start of the timed region (host wall clock, the clock nvidia-smi stamps with)."""
        self.t0 = time.time()

    def end(self) -> None:
        self.t1 = time.time()

    def stop(self) -> dict | None:
        if self.p is None:
            return None
        time.sleep(0.25)  # one more sample after the window
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        txt = Path(self.f.name).read_text()
        os.unlink(self.f.name)
        from datetime import datetime

        rows = []
        for r in txt.splitlines():
            c = [x.strip() for x in r.split(",")]
            try:
                t = datetime.strptime(c[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((t, float(c[2]), float(c[3]), float(c[4]), c[5:9]))
            except (ValueError, IndexError):
                continue
        if not rows:
            return None
        t0, t1 = self.t0 or rows[0][0], self.t1 or rows[-1][0]
        inside = [r for r in rows if t0 <= r[0] <= t1] or [min(rows, key=lambda r: abs(r[0] - t1))]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({nm for r in inside for nm, v in zip(names, r[4]) if v.lower() == "active"})
        power = [(r[0], r[3]) for r in rows]
        dedup = []
        for t, w in power:  # strictly increasing timestamps for window_average
            if not dedup or t > dedup[-1][0]:
                dedup.append((t, w))
        try:
            avg_w = window_average(dedup, t0, t1) if t1 > t0 else dedup[-1][1]
        except ValueError:
            avg_w = None
        return {"gpu": self.idx, "sm_mhz": float(np.median([r[1] for r in inside])),
                "sm_max_mhz": max(r[2] for r in inside), "reasons": reasons, "samples": len(inside),
                "power_w_window_avg": avg_w, "window_s": t1 - t0}


def dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def cpu_oracle_pair_ms(T: int, nfld_sample: int, nfld_full: int, pairs: int = 1, warm: int = 0):
    """Time the CPU oracle (NumPy/SciPy port, all host threads) on a bounded
    sample of the workload and scale linearly in the field count."""
    from oracle.sht_oracle import SHTransformOracle, random_spectral

    o = SHTransformOracle(T, nfld=nfld_sample, workers=os.cpu_count())
    a = random_spectral(T, nfld_sample)
    for _ in range(warm):
        o.dir_trans(o.inv_trans(a))
    times = []
    for _ in range(pairs):
        t0 = time.perf_counter()
        o.dir_trans(o.inv_trans(a))
        times.append((time.perf_counter() - t0) * 1e3)
    per = float(np.mean(times))
    return per * nfld_full / nfld_sample, per, times


def traffic_per_launch(kernel: str, T: int, nfld: int, P: int, mode: str):
    """DRAM bytes (read + write) per launch of `kernel` from an `ncu --set full` capture of this exact
    configuration (profiles/traffic.json, keyed "TCo{T}_nfld{nfld}_P{P}_{mode}"), else None."""
    f = ROOT / "profiles" / "traffic.json"
    if f.exists():
        try:
            return json.loads(f.read_text()).get(f"TCo{T}_nfld{nfld}_P{P}_{mode}", {}).get(kernel)
        except Exception:
            return None
    return None


def config_of(args) -> dict:
    """The workload keys both arms report (identical, so the driver can match them)."""
    T, nf = args.truncation, args.nfld
    return {"workload": f"TCo{T} inverse+direct pair, {nf} fields", "truncation": T, "nfld": nf,
            "grid": "octahedral"}


def run_reference(args):
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    T, nf, ns = args.truncation, args.nfld, args.cpu_fields
    from oracle.sht_oracle import SHTransformOracle, random_spectral

    o = SHTransformOracle(T, nfld=ns, workers=cores)
    a = random_spectral(T, ns)
    warm = min(args.warmup, 1)  # one warm-up pair: the CPU path has no caches worth more
    for _ in range(warm):
        o.dir_trans(o.inv_trans(a))
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.dir_trans(o.inv_trans(a))
    per_sample = (time.perf_counter() - t0) * 1e3 / args.steps
    value = per_sample * nf / ns
    sample = (f"TCo{T}, {ns} of {nf} fields per inv+dir pair (CPU oracle oracle/sht_oracle.py: NumPy BLAS "
              f"Legendre GEMMs + scipy.fft ring FFTs, workers={cores}), time scaled x{nf}/{ns} (linear in fields); "
              f"{warm} warm-up pair(s)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "lscpu": lscpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference (haloflow) has no transform code (SPEC.md:20); its CPU path is the oracle port",
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1908_06097_b200 import SHTransform

    refuse_debug()
    rank, world, local = dist_setup()
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    group = dist.group.WORLD if world > 1 else None
    T, nf = args.truncation, args.nfld
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.perf_counter()
    gp = tuple(int(x) for x in args.gp_layout.split(",")) if args.gp_layout else None
    sh = SHTransform(T, nfld=nf, group=group, profile=True, recompute_legendre=args.recompute_legendre,
                     gp_layout=gp)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0

    g = torch.Generator(device=dev)
    g.manual_seed(T * 1000 + rank)
    spec = torch.randn(nf, sh.nspec_local, dtype=torch.float64, device=dev, generator=g) / np.sqrt(2.0)
    if 0 in sh.m_list:  # Im a_n^0 = 0 (m = 0 is the first local wavenumber when present)
        spec[:, 1: 2 * (T + 1): 2] = 0.0
    grid = torch.empty(nf, sh.npts_grid, dtype=torch.float64, device=dev)
    spec2 = torch.empty_like(spec)

    def pair():
        sh.inv_trans(spec, out=grid)
        sh.dir_trans(grid, out=spec2)

    clk = Clocks(local)  # every rank samples its own GPU; started before the warm-up (NVML start-up)
    for _ in range(args.warmup):
        pair()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk.mark()
    e0.record()
    for _ in range(args.steps):
        pair()
    e1.record()
    torch.cuda.synchronize()
    clk.end()
    if world > 1:
        dist.barrier()
    clk_local = clk.stop()
    if world > 1:
        allc = [None] * world
        dist.all_gather_object(allc, clk_local)
    else:
        allc = [clk_local]
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms_local, world)
    ph = sh.phase_ms(min(args.steps, 64))
    work = sh.work()
    launches = sh.kernel_launches()

    # end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # each step: one host batch in (H2D), its inverse + direct pair, the result
        # out (D2H); SHTransform.pairs_pipelined overlaps the copies of batches
        # i+1 / i-1 with the transforms of batch i (PCIe is full duplex)
        h = np.ascontiguousarray(spec.cpu().numpy())
        host_in = [torch.from_numpy(h.copy()).pin_memory() for _ in range(2)]
        host_out = [torch.empty(spec.shape, dtype=torch.float64).pin_memory() for _ in range(2)]
        sh.pairs_pipelined(host_in, host_out)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record()
        sh.pairs_pipelined([host_in[i % 2] for i in range(args.steps)], [host_out[i % 2] for i in range(args.steps)])
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        nbytes = spec.numel() * 8
        e2e = {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "path": "SHTransform.pairs_pipelined (C-ABI inv_trans/dir_trans) with every step's spectral batch copied in from pinned host memory and its result copied back, copies overlapped with the neighbouring steps' transforms"}

    pk = peaks()
    # per-rank phase times (max over ranks = the critical path)
    leg_ms = max_over_ranks(ph["inv_legendre"] + ph["dir_legendre"], world)
    fft_ms = max_over_ranks(ph["inv_fft"] + ph["dir_fft"], world)
    a2a_ms = max_over_ranks(ph["inv_alltoall"] + ph["dir_alltoall"], world)
    F_leg = max_over_ranks(work["legendre_flops"], world)
    B_fft = max_over_ranks(work["fft_bytes"], world)
    B_a2a = max_over_ranks(work["a2a_bytes"], world)
    t_leg_roof = F_leg / (pk["fp64_tflops"] * 1e12) * 1e3
    t_fft_roof = B_fft / (pk["hbm_gbs"] * 1e9) * 1e3
    transport = sh.transport
    row_layout = sh.row_layout
    t_a2a_roof = B_a2a / (pk["nvlink_gbs"] * 1e9) * 1e3 if world > 1 else 0.0
    p2p = transport == "p2p"
    # p2p: the NVLink stores run inside the producing kernels (leg_inv -> ring owners, fft_g2f -> m
    # owners), so each of those is bounded by max(its own work / its peak, its NVLink bytes / 770 GB/s)
    # (B200_PROFILING.md fused compute+collective roofline); nccl: the transfer is a phase of its own
    t_a2a_dir = t_a2a_roof / 2
    t_roof = (max(t_leg_roof / 2, t_a2a_dir if p2p else 0.0) + t_leg_roof / 2 +
              t_fft_roof / 2 + max(t_fft_roof / 2, t_a2a_dir if p2p else 0.0) + (0.0 if p2p else t_a2a_roof))

    def mx(v):
        return max_over_ranks(v, world)

    mode = "recompute" if args.recompute_legendre else "table"
    nvl = B_a2a / 2 if p2p else 0.0  # bytes one rank stores into its peers per direction
    kern = {
        "leg_inv_kernel": ("tensor", mx(ph["inv_legendre"]), F_leg / 2, 1e12, "TFLOP/s", pk["fp64_tflops"],
                           pk["fp64_src"], f"{F_leg / 2:.4e} FP64 flop (4*NFLD*sum_m NDGLU(m)(T-m+1) per direction)",
                           nvl),
        "leg_dir_kernel": ("tensor", mx(ph["dir_legendre"]), F_leg / 2, 1e12, "TFLOP/s", pk["fp64_tflops"],
                           pk["fp64_src"], f"{F_leg / 2:.4e} FP64 flop", 0.0),
        "fft_f2g": ("hbm", mx(ph["inv_fft"]), B_fft / 2, 1e9, "GB/s", pk["hbm_gbs"], pk["hbm_src"],
                    f"{B_fft / 2:.4e} B (grid 8 B x 2 N_i + Fourier rows 32 B x (M_i+1), per field and ring pair)",
                    0.0),
        "fft_g2f": ("hbm", mx(ph["dir_fft"]), B_fft / 2, 1e9, "GB/s", pk["hbm_gbs"], pk["hbm_src"],
                    f"{B_fft / 2:.4e} B", nvl),
    }
    rooflines = {}
    for name, (bound, t_ms, amount, scale, unit, peak, src, per, nvbytes) in kern.items():
        ach = amount / scale / (t_ms * 1e-3) if t_ms > 0 else 0.0
        r = {"bound": bound, "kernel": name, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
             "traffic": traffic_per_launch(name, T, nf, world, mode), "ms": t_ms, "peak_src": src,
             "per_launch": per}
        if nvbytes > 0:  # fused compute + NVLink stores: the slower of the two ceilings
            t_work = amount / scale / peak * 1e3
            t_nvl = nvbytes / (pk["nvlink_gbs"] * 1e9) * 1e3
            r["fused_nvlink"] = {"nvlink_bytes": nvbytes, "t_work_ms": t_work, "t_nvlink_ms": t_nvl,
                                 "t_roof_ms": max(t_work, t_nvl), "frac": max(t_work, t_nvl) / t_ms if t_ms else None,
                                 "nvlink_gbs_achieved": nvbytes / (t_ms * 1e-3) / 1e9 if t_ms else None}
        rooflines[name] = r
    dom = max(rooflines, key=lambda k: rooflines[k]["ms"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        full, per, _ = cpu_oracle_pair_ms(T, args.cpu_fields, nf, pairs=1, warm=0)
        cpu = {"value": full, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"TCo{T}, {args.cpu_fields} of {nf} fields, one inv+dir pair of the CPU oracle "
                         f"(NumPy BLAS + scipy.fft, all host threads) = {per:.1f} ms, scaled x{nf}/{args.cpu_fields}",
               "lscpu": lscpu()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(args),
            "layout": {"parallelism": f"m/ring-pair sharded x{world}, transposition: {transport}",
                       "fourier_rows": row_layout,
                       "transport_env": os.environ.get("SHT_TRANSPORT", "p2p (default)"),
                       "gp_layout": args.gp_layout or "ring pairs (no grid-point transposition)",
                       "legendre": "recomputed per transform" if args.recompute_legendre else "stored table",
                       "l2": (f"no flush: inputs larger than L2 (spectral {spec.numel() * 8 / 1e9:.2f} GB, grid "
                              f"{grid.numel() * 8 / 1e9:.2f} GB per rank vs 126 MB L2)")},
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "roofline": rooflines[dom],
            "rooflines": rooflines,
            "combined_roofline": {
                "t_roof_ms": t_roof, "frac": t_roof / ms, "legendre_roof_ms": t_leg_roof,
                "fft_roof_ms": t_fft_roof, "a2a_roof_ms": t_a2a_roof, "transport": transport,
                "phases_ms": {"legendre": leg_ms, "fft": fft_ms, "alltoall": a2a_ms},
                "phase_frac": {"legendre_fp64": t_leg_roof / leg_ms if leg_ms else None,
                               "fft_hbm": t_fft_roof / fft_ms if fft_ms else None,
                               "alltoall_nvlink": (t_a2a_roof / a2a_ms) if a2a_ms else None},
                "peaks": pk,
            },
            "phases_ms": ph,
            "setup_s": setup_s,
            "cpu_baseline": cpu,
            "clocks": ({"sm_mhz": float(np.median([c["sm_mhz"] for c in allc if c])),
                        "sm_max_mhz": max(c["sm_max_mhz"] for c in allc if c),
                        "reasons": sorted({r for c in allc if c for r in c["reasons"]}),
                        "per_gpu": allc} if any(allc) else None),
            # per-GPU NVML power, each averaged over the timed window with the
            # reference's window_average (energy.py:83-111), summed over GPUs x ms per pair
            # (energy_per_step, energy.py:114-123)
            "energy": ({"j_per_pair": sum(c["power_w_window_avg"] for c in allc) * ms * 1e-3,
                        "power_w_per_gpu": [c["power_w_window_avg"] for c in allc],
                        "basis": "per-GPU nvidia-smi power.draw, window_average over the timed region"}
                       if all(c and c.get("power_w_window_avg") for c in allc) else None),
        }
        print(json.dumps(line), flush=True)
    sh.close()  # collective: every rank releases its plan after the peers are done with it
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
