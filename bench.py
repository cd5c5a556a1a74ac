"""Benchmark of the log-polar Radon transform R and back-projection R#
(BASELINE.json metric: "R and R# slices/sec at N=2048 (1/2/4/8 B200),
% HBM roofline, vs host-CPU ref").

A step = one R followed by one R# (the normal operator R# R of iterative
reconstruction) over a batch of B slices per GPU of the N=2048 stack
(3072 angles, M=3 sectors). `value` counts slices that went through both
operators per second over all ranks (weak scaling: B fixed per GPU, slices
sharded, no collective on the data path). Inputs are device-resident
synthetic Shepp-Logan / random-disc slices, B * 16.8 MB > L2 per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun every rank runs its shard; rank 0 prints one JSON line with
the max-over-ranks device time. `--impl reference` times the CPU
restatement of the reference path (oracle/, the reference's lp_ops is
unimplemented upstream) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "R and R# slices/sec at N=2048 (1/2/4/8 B200), % HBM roofline, vs host-CPU ref"
UNIT = "slices/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=16, help="slices per GPU per step")
    ap.add_argument("--plan", choices=["smooth", "default"], default="smooth",
                    help="smooth: N_rho rounded up to a 7-smooth FFT length; default: minimal N_rho")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-reps", type=int, default=5)
    return ap.parse_args()


def world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def geometry(args):
    import paper_1506_00014_b200 as lp

    n_rho = lp.smooth_n_rho(args.n) if args.plan == "smooth" else 0
    return lp.sampling_plan(args.n, 3, 0, n_rho)


def config(args, g, n_gpus):
    return {
        "workload": f"N={g.N} stack, {g.n_theta} angles, M={g.M}, step = R then R# on {args.batch} slices/GPU",
        "N": g.N, "n_theta": g.n_theta, "M": g.M, "n_rho": g.n_rho, "plan": args.plan,
        "global_batch": args.batch * n_gpus, "parallelism": f"slices sharded dp{n_gpus}",
        "l2": "inputs larger than L2 (batch x 16.8 MB per step)",
        "inputs": "alternating modified Shepp-Logan and smooth random-disc slices, generated on device",
    }


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names[1:], parts[3:]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def gpu_index(local_rank: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v for v in vis.split(",") if v.strip()]
        if local_rank < len(ids) and ids[local_rank].strip().isdigit():
            return int(ids[local_rank])
    return local_rank


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# stage name (lpr_gpu_profile_stages) -> the kernel(s) that implement it
STAGE_KERNELS = {
    "prefilter_2d": ("k_prefilter_2d_iir",),
    "prefilter_sino": ("k_prefilter_sino_iir",),
    "rho_pass": ("k_rho_stream", "k_rho_pass", "k_rho_pad"),
    "radon_out": ("k_radon_out_b", "k_radon_out"),
}


def ncu_lsu_pct(stage: str):
    """L1/LSU data-pipe utilisation (% of peak) of `stage`'s kernel from the
    latest committed ncu capture (profiles/*/ncu_dram_bytes.json), or None."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_dram_bytes.json")), key=os.path.getmtime)
    for path in reversed(files):
        try:
            with open(path) as f:
                per = json.load(f).get("lsu_wavefronts_pct", {})
        except Exception:
            continue
        kernels = STAGE_KERNELS.get(stage, ("k_" + stage,))
        for name, v in per.items():
            if any(name == k or name.startswith(k + "<") for k in kernels):
                return v
    return None


def ncu_traffic(stage: str, slices: int):
    """dram__bytes_read + dram__bytes_write of `stage`'s kernel from the latest
    committed `ncu --set full` capture (profiles/*/ncu_dram_bytes.json, per
    slice), scaled to one launch of `slices` slices; None if not captured."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_dram_bytes.json")), key=os.path.getmtime)
    for path in reversed(files):
        try:
            with open(path) as f:
                per = json.load(f)["per_slice_bytes"]
        except Exception:
            continue
        kernels = STAGE_KERNELS.get(stage, ("k_" + stage,))
        for name, b in per.items():
            if any(name == k or name.startswith(k + "<") for k in kernels):
                return b * slices
    return None


def pcie_ceiling(h_img, d_img, d_sino, h_sino, nbytes_img, nbytes_sino, slices):
    """Host<->device copy bandwidth, both directions at once (the e2e step moves
    images in and sinograms out for R, the reverse for R#), and the e2e
    throughput the link alone would allow: R phase max(H2D img, D2H sino) +
    R# phase max(H2D sino, D2H img) when the calls run one after the other,
    (img + sino) per direction when they are pipelined."""
    import torch

    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    reps = 2
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d_img.copy_(h_img, non_blocking=True)
        with torch.cuda.stream(s2):
            h_sino.copy_(d_sino, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    gbs = max(nbytes_img, nbytes_sino) / dt / 1e9
    step = 2 * max(nbytes_img, nbytes_sino) / (gbs * 1e9)
    # pipelined (R of step k beside R# of step k-1): each direction carries
    # one image and one sinogram per slice per step
    step_pipe = (nbytes_img + nbytes_sino) / (gbs * 1e9)
    return {"link_duplex_gbs": gbs, "link_bound_value": slices / step, "link_bound_pipelined_value": slices / step_pipe}


# ------------------------------------------------------------------ CPU legs
def cpu_sample(g, zeta, zeta_bp, slices: int = 1):
    """R then R# of `slices` slices through the oracle (fp64 CPU restatement,
    OpenMP over all host threads). Returns seconds per slice."""
    from oracle import lpo

    p = lpo.make_plan(g.N, g.M, g.n_theta, g.n_rho)
    f = lpo.phantom_image(g.N)
    t = time.perf_counter()
    for _ in range(slices):
        s = lpo.fast_radon(p, zeta, f)
        lpo.fast_backprojection(p, zeta_bp, s)
    return (time.perf_counter() - t) / slices


def run_reference(args):
    rank, ws, _ = world()
    if rank != 0:
        return
    import paper_1506_00014_b200 as lp

    g = geometry(args)
    z, zb = lp.zeta_spectrum(g), lp.zeta_bp_spectrum(g)  # plan constants, excluded from timing
    cores = os.cpu_count()
    warm = min(args.warmup, 1)
    est = 0.0
    for _ in range(warm):
        est = cpu_sample(g, z, zb)
    steps = args.steps
    if est > 0:
        steps = max(1, min(args.steps, int(150.0 / est)))
    t = time.perf_counter()
    for _ in range(steps):
        cpu_sample(g, z, zb)
    dt = (time.perf_counter() - t) / steps
    value = 1.0 / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": steps,
        "warmup": warm, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config(args, g, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": "1 slice (R then R#) per step at the bench plan; the reference's lp_ops is "
                                   "unimplemented upstream, so this is the fp64 oracle restatement composed of "
                                   "blocks verified bit-identical to the reference's compiled geometry/bspline/"
                                   "kernel code, OpenMP over all host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1506_00014_b200 as lp
    from paper_1506_00014_b200 import phantoms, roofline, sharding
    from paper_1506_00014_b200.sharding import stack_shard

    rank, ws, local = world()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    g = geometry(args)
    z, zb = lp.zeta_spectrum(g, device=local), lp.zeta_bp_spectrum(g, device=local)  # plan constants (GPU fp64)
    B = args.batch
    plan = lp.RadonPlan(g, z, zb, max_batch=B, device=local)
    start, count = stack_shard(B * ws, ws, rank)  # this rank's slices of the stack (weak scaling)
    assert count == B
    imgs = phantoms.stack(g.N, B, seed0=0x5EED + start, device=dev)
    sino = torch.empty(B, g.n_theta, g.N, device=dev)
    back = torch.empty(B, g.N, g.N, device=dev)
    stream = torch.cuda.current_stream(dev)
    h = plan.handle
    L = lp._lib.lib()
    sp = stream.cuda_stream

    def step():
        lp._lib.check(L.lpr_gpu_radon(h, imgs.data_ptr(), sino.data_ptr(), B, sp))
        lp._lib.check(L.lpr_gpu_backproject(h, sino.data_ptr(), back.data_ptr(), B, sp))

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        return sharding.max_over_ranks(x, device=dev)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches0 = plan.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu_index(local)) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = plan.launch_count() - launches0
    ms_step = ms / args.steps
    value = ws * B * args.steps / (ms / 1e3)

    # R-only / R#-only throughput (same buffers, device events)
    def timed(fn, n=5):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b)) / n

    ms_r = timed(lambda: lp._lib.check(L.lpr_gpu_radon(h, imgs.data_ptr(), sino.data_ptr(), B, sp)))
    ms_b = timed(lambda: lp._lib.check(L.lpr_gpu_backproject(h, sino.data_ptr(), back.data_ptr(), B, sp)))

    # end to end through the public host API: pinned host slices in, H2D,
    # R, D2H sinogram, then H2D sinogram, R#, D2H image, every step.
    h_img = torch.empty(B, g.N, g.N, pin_memory=True)
    h_img.copy_(imgs.cpu())
    h_sino = torch.empty(B, g.n_theta, g.N, pin_memory=True)
    h_back = torch.empty(B, g.N, g.N, pin_memory=True)
    hp = (h_img.data_ptr(), h_sino.data_ptr(), h_back.data_ptr())

    def e2e_step():
        lp._lib.check(L.lpr_gpu_radon_host(h, hp[0], hp[1], B))
        lp._lib.check(L.lpr_gpu_backproject_host(h, hp[1], hp[2], B))

    e2e_step()
    e2e_steps = max(2, min(args.steps, 5))
    barrier()
    t = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = max_over_ranks((time.perf_counter() - t) / e2e_steps)
    e2e_seq_value = ws * B / e2e_s

    # The same job software-pipelined across steps through the same public
    # calls: one host thread runs R of steps 0..K-1 (plan 1), a second runs R#
    # of steps 0..K-1 (plan 2), R# of step k starting once R of step k has
    # returned its sinograms (two pinned sinogram buffers; R of step k+2 waits
    # for R# of step k to release its buffer). The host link then carries
    # images in + sinograms out of R and sinograms in + images out of R# at the
    # same time (a lone R call is D2H-bound, a lone R# call H2D-bound), and the
    # calls' own fill/drain overlaps the other thread's work. Every step still
    # copies all of its inputs from pinned host memory and its results back;
    # the wall clock spans the first R's start to the last R#'s end (K steps,
    # the pipeline fill and drain included).
    plan2 = lp.RadonPlan(g, z, zb, max_batch=B, device=local)
    h2 = plan2.handle
    h_sino2 = torch.empty(B, g.n_theta, g.N, pin_memory=True)
    sino_bufs = (hp[1], h_sino2.data_ptr())

    def e2e_pipelined(K):
        done_r = [threading.Event() for _ in range(K)]
        done_b = [threading.Event() for _ in range(K)]
        errors = []

        def r_loop():
            try:
                for k in range(K):
                    if k >= 2:
                        done_b[k - 2].wait()
                    lp._lib.check(L.lpr_gpu_radon_host(h, hp[0], sino_bufs[k % 2], B))
                    done_r[k].set()
            except Exception as e:  # surfaced below; unblock the other thread
                errors.append(e)
                for ev in done_r:
                    ev.set()

        def b_loop():
            try:
                for k in range(K):
                    done_r[k].wait()
                    if errors:
                        return
                    lp._lib.check(L.lpr_gpu_backproject_host(h2, sino_bufs[k % 2], hp[2], B))
                    done_b[k].set()
            except Exception as e:
                errors.append(e)
                for ev in done_b:
                    ev.set()

        threads = [threading.Thread(target=r_loop), threading.Thread(target=b_loop)]
        t0 = time.perf_counter()
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        dt = time.perf_counter() - t0
        if errors:
            raise errors[0]
        return dt / K

    e2e_pipelined(2)  # warm-up
    barrier()
    e2e_pipe_k = max(4, min(2 * args.steps, 8))
    e2e_pipe_s = max_over_ranks(e2e_pipelined(e2e_pipe_k))
    plan2.close()
    e2e_value = ws * B / e2e_pipe_s
    nbytes_img, nbytes_sino = B * g.N * g.N * 4, B * g.n_theta * g.N * 4
    link = pcie_ceiling(h_img, imgs, sino, h_sino, nbytes_img, nbytes_sino, ws * B)

    # per-kernel durations measured live on the plan's stream; roofline of the
    # dominant kernel against the measured HBM copy bandwidth
    prof_r = roofline.profile_stages(plan, "radon", imgs.data_ptr(), sino.data_ptr(), B, args.profile_reps)
    prof_b = roofline.profile_stages(plan, "backproject", sino.data_ptr(), back.data_ptr(), B, args.profile_reps)
    by_r = roofline.stage_bytes(g, "radon", B)
    by_b = roofline.stage_bytes(g, "backproject", B)
    stages = {}
    for op, prof, by in (("R", prof_r, by_r), ("R#", prof_b, by_b)):
        for k, v in prof.items():
            stages[f"{op}:{k}"] = {"ms": v, "bytes": by[k], "GBps": by[k] / (v * 1e-3) / 1e9}
    total = sum(s["ms"] for s in stages.values())
    dom_name, dom = max(stages.items(), key=lambda kv: kv[1]["ms"])
    peak, peak_kind = measured_peak()
    traffic = ncu_traffic(dom_name.split(":", 1)[1], B)
    for s in stages.values():
        s["share"] = s["ms"] / total
        s["frac"] = s["GBps"] / peak

    result = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            try:
                sec = cpu_sample(g, z, zb)
                cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                       "sample": "1 slice of the same workload (Shepp-Logan, R then R#) through the fp64 oracle "
                                 "restatement with OpenMP on all host threads; plan constants excluded"}
            except Exception as e:  # the CPU leg is a reported baseline, not the product
                cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                       "sample": f"unavailable: {e}"}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config(args, g, ws),
            "radon_slices_per_s": ws * B / (ms_r / 1e3), "backproject_slices_per_s": ws * B / (ms_b / 1e3),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes_img + nbytes_sino,
                    "d2h_bytes_per_step": nbytes_sino + nbytes_img,
                    "how": "lpr_gpu_radon_host of steps 0..K-1 on one host thread / plan and "
                           "lpr_gpu_backproject_host of steps 0..K-1 (each on its step's sinograms) on a second, "
                           "pipelined; pinned host buffers, every copy inside the wall clock, fill and drain included",
                    "pipelined_steps": e2e_pipe_k,
                    "sequential_value": e2e_seq_value, **link},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": dom["GBps"], "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": dom["GBps"] / peak,
                         "traffic": traffic, "share_of_step": dom["share"],
                         "l1_lsu_pct_ncu": ncu_lsu_pct(dom_name.split(":", 1)[1]),
                         "algorithmic_bytes_per_launch": dom["bytes"], "ms_per_launch": dom["ms"]},
            "stages": stages,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(result), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    plan.close()
    return result


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
