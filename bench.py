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

`--gpus N` > 1 outside torchrun re-executes the bench under
`torch.distributed.run` with N ranks (one per GPU, NCCL). Every rank runs its
shard; rank 0 prints one JSON line with the max-over-ranks device time, and
`gathered` times the same step followed by a grouped NCCL send/recv of every
rank's sinograms to rank 0 (the optional final gather).
`--dry-run` runs that rank / shard / gather plumbing with gloo on CPU tensors
(no GPU work, no measurement; the CPU test of the multi-rank path).
`--impl reference` times the CPU restatement of the reference path
(oracle/, the reference's lp_ops is unimplemented upstream) on the host
cores, rank 0 only; it loads nothing from the product package.
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
    ap.add_argument("--size", dest="n", type=int, default=2048, help="image size N")
    ap.add_argument("--batch", type=int, default=16, help="slices per GPU per step")
    ap.add_argument("--plan", choices=["smooth", "default"], default="smooth",
                    help="smooth: N_rho rounded up to a 7-smooth FFT length; default: minimal N_rho")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-reps", type=int, default=5)
    ap.add_argument("--dry-run", action="store_true", help="gloo on CPU: rank/shard/gather plumbing only")
    ap.add_argument("--no-default-plan", action="store_true", help="skip the default-plan (minimal N_rho) row")
    ap.add_argument("--stack", type=int, default=2048,
                    help="config 4: slices of the whole stack sharded over the ranks (0 skips the row)")
    return ap.parse_args()


def relaunch(args) -> int:
    """--gpus N outside torchrun: run this script under torch.distributed.run
    with N ranks (127.0.0.1 rendezvous) and return its exit code."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def smooth_at_least(n: int) -> int:
    """Smallest length >= n whose factors are all in {2, 3, 5, 7}."""
    while True:
        m = n
        for f in (2, 3, 5, 7):
            while m % f == 0:
                m //= f
        if m == 1:
            return n
        n += 1


def geometry(args, plan=None):
    import paper_1506_00014_b200 as lp

    plan = plan or args.plan
    n_rho = lp.smooth_n_rho(args.n) if plan == "smooth" else 0
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


def _ncu_capture():
    """The latest committed ncu summary (profiles/*/ncu_kernels.json): per kernel
    the batch of the captured launch, its dram__bytes_read + write and its
    L1/LSU data-pipe utilisation."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_kernels.json")))
    for path in reversed(files):
        try:
            with open(path) as f:
                return json.load(f), os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def ncu_for(stage: str, batch: int):
    """(traffic bytes per launch of `batch` slices, L1/LSU %, source) of the
    kernel implementing `stage`, from one `ncu --set full` capture of the
    bench-size launch; (None, None, None) when not captured."""
    cap, src = _ncu_capture()
    if not cap:
        return None, None, None
    kernels = STAGE_KERNELS.get(stage, ("k_" + stage,))
    for name, rec in cap.get("kernels", {}).items():
        if any(name == k or name.startswith(k + "<") for k in kernels):
            return rec["dram_bytes"] * batch / rec["batch"], rec.get("lsu_pct"), src
    return None, None, None


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
def oracle_plan(args, plan=None):
    """The bench plan built by the oracle alone (no product code loaded)."""
    from oracle import lpo

    p = lpo.make_plan(args.n, 3)
    if (plan or args.plan) == "smooth":
        p = lpo.make_plan(args.n, 3, 0, smooth_at_least(p.n_rho))
    return p


def cpu_sample(p, zeta, zeta_bp, slices: int = 1):
    """R then R# of `slices` slices through the oracle (fp64 CPU restatement,
    OpenMP over all host threads). Returns seconds per slice."""
    from oracle import lpo

    f = lpo.phantom_image(p.N)
    t = time.perf_counter()
    for _ in range(slices):
        s = lpo.fast_radon(p, zeta, f)
        lpo.fast_backprojection(p, zeta_bp, s)
    return (time.perf_counter() - t) / slices


CPU_SAMPLE = ("1 slice (Shepp-Logan, R then R#) per step of the same N=2048 plan; the reference's lp_ops is "
              "unimplemented upstream, so this is the fp64 oracle restatement composed of blocks verified "
              "bit-identical to the reference's compiled geometry/bspline/kernel code, OpenMP over all host "
              "threads; plan constants (spectra) excluded")


def run_reference(args):
    """The reference arm: oracle/ only (lpo.make_plan, lpo.spectrum, Algorithms
    1-2 in fp64), rank 0 of N; the other ranks exit without work."""
    rank, ws, _ = world()
    if rank != 0:
        return
    # all host threads (torchrun exports OMP_NUM_THREADS=1 to every rank; the
    # oracle's OpenMP runtime reads it when oracle/liblpo.so is first loaded)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
    from oracle import lpo

    p = oracle_plan(args)
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)  # plan constants, excluded from timing
    cores = os.cpu_count()
    warm = max(args.warmup, 3)
    for _ in range(warm):
        cpu_sample(p, z, zb)
    t = time.perf_counter()
    for _ in range(args.steps):
        cpu_sample(p, z, zb)
    dt = (time.perf_counter() - t) / args.steps
    value = 1.0 / dt
    # the same plan and metric as the GPU arm; a CPU step is one slice (the GPU arm's is 16 per GPU)
    ref_cfg = config(args, p, ws)
    ref_cfg["global_batch"] = 1
    ref_cfg["workload"] = (f"N={p.N} stack, {p.n_theta} angles, M={p.M}, step = R then R# on 1 slice "
                           "(CPU; the GPU arm's step is 16 slices per GPU)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": warm, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": ref_cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": CPU_SAMPLE,
                         "slices_per_step": 1},
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
    if ws != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws}")
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

    # the same step followed by the final gather of every rank's sinograms to
    # rank 0 (grouped NCCL send/recv over NVLink; SURVEY.md §8(e) reports it as
    # a separate row: rank 0's ingress bounds it, the sharded value does not)
    gather_out = torch.empty(ws * B, g.n_theta, g.N, device=dev) if (rank == 0 and ws > 1) else None

    def gathered_step():
        step()
        sharding.gather_to_root(sino, 0, gather_out)

    for _ in range(2):
        gathered_step()
    torch.cuda.synchronize()
    barrier()
    ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ga.record(stream)
    g_steps = max(2, min(args.steps, 10))
    for _ in range(g_steps):
        gathered_step()
    gb.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_g = max_over_ranks(ga.elapsed_time(gb)) / g_steps
    sino_bytes = B * g.n_theta * g.N * 4
    gathered = {"value": ws * B / (ms_g / 1e3), "unit": UNIT, "ms_per_step": ms_g, "steps": g_steps,
                "bytes_to_rank0_per_step": (ws - 1) * sino_bytes,
                "how": "step + torch batch_isend_irecv (grouped ncclSend/ncclRecv) of every rank's "
                       f"{B} sinograms to rank 0, device events, max over ranks"}
    del gather_out

    # config 4 (BASELINE.json): the whole 2048-slice stack sharded over the
    # ranks, each rank's contiguous shard device resident (distinct slices,
    # 34 GB at one GPU), R then R# chunk by chunk (B slices per launch)
    stack = None
    if args.stack > 0:
        s_start, s_count = stack_shard(args.stack, ws, rank)
        stack_in = phantoms.stack(g.N, s_count, seed0=0x5EED + s_start, device=dev) if s_count else None
        torch.cuda.synchronize()

        def stack_job():
            for c0 in range(0, s_count, B):
                nb = min(B, s_count - c0)
                x = stack_in[c0:c0 + nb]
                lp._lib.check(L.lpr_gpu_radon(h, x.data_ptr(), sino.data_ptr(), nb, sp))
                lp._lib.check(L.lpr_gpu_backproject(h, sino.data_ptr(), back.data_ptr(), nb, sp))

        barrier()
        sa, sb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sa.record(stream)
        stack_job()
        sb.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_stack = max_over_ranks(sa.elapsed_time(sb))
        stack = {"slices": args.stack, "slices_per_rank": s_count, "chunk": B, "ms": ms_stack,
                 "value": args.stack / (ms_stack / 1e3), "unit": UNIT,
                 "how": "the whole stack sharded contiguously over the ranks, each shard device resident "
                        "(distinct Shepp-Logan / random-disc slices), R then R# per chunk of B slices, "
                        "device events, max over ranks, one pass (no warm-up beyond the main run's)"}
        del stack_in

    # R-only / R#-only throughput (same buffers, device events)
    def timed(fn, n=5, warm=1):
        for _ in range(warm):
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
    # the callers next to the path: FBP (cosine filter, c_norm R#(filter g)) and EM
    # iterations (R, ratio, R#, update; g >= 0) on the same stack, device time per slice
    ms_fbp = timed(lambda: lp._lib.check(L.lpr_gpu_fbp(h, 2, sino.data_ptr(), back.data_ptr(), B, sp)))
    g_pos = sino.clamp_min(0)
    em_iters = 3
    ms_em = timed(lambda: lp._lib.check(L.lpr_gpu_em(h, g_pos.data_ptr(), back.data_ptr(), B, em_iters, 1, None, sp)),
                  n=2) / em_iters
    del g_pos

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
    sep_value = ws * B / e2e_pipe_s

    # The step itself through the one-call public API for it,
    # lpr_gpu_radon_backproject_host (R then R# of the same slices: images in,
    # sinograms and back-projections out, the sinograms not re-uploaded), steps
    # alternating between two host threads / plans so one call's pipeline fill
    # and drain overlap the other's. Every step copies its images in and both
    # results out inside the wall clock.
    h_sino_b = torch.empty(B, g.n_theta, g.N, pin_memory=True)
    h_back_b = torch.empty(B, g.N, g.N, pin_memory=True)
    outs = ((hp[1], hp[2]), (h_sino_b.data_ptr(), h_back_b.data_ptr()))

    def e2e_normal(K):
        errors = []

        def loop(t):
            try:
                for k in range(t, K, 2):
                    lp._lib.check(L.lpr_gpu_radon_backproject_host((h, h2)[t], hp[0], outs[t][0], outs[t][1], B))
            except Exception as e:
                errors.append(e)

        threads = [threading.Thread(target=loop, args=(t,)) for t in (0, 1)]
        t0 = time.perf_counter()
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        dt = time.perf_counter() - t0
        if errors:
            raise errors[0]
        return dt / K

    e2e_normal(2)  # warm-up
    barrier()
    e2e_norm_s = max_over_ranks(e2e_normal(e2e_pipe_k))
    plan2.close()
    e2e_value = ws * B / e2e_norm_s
    nbytes_img, nbytes_sino = B * g.N * g.N * 4, B * g.n_theta * g.N * 4
    link = pcie_ceiling(h_img, imgs, sino, h_sino, nbytes_img, nbytes_sino, ws * B)

    # per-kernel durations measured live on the plan's stream; roofline of the
    # dominant kernel against the measured HBM copy bandwidth
    prof_r = roofline.profile_stages(plan, "radon", imgs.data_ptr(), sino.data_ptr(), B, args.profile_reps)
    prof_b = roofline.profile_stages(plan, "backproject", sino.data_ptr(), back.data_ptr(), B, args.profile_reps)
    peak, peak_kind = measured_peak()
    stages = {}
    for op, name, prof in (("R", "radon", prof_r), ("R#", "backproject", prof_b)):
        by, comp = roofline.stage_bytes(g, name, B), roofline.compulsory_bytes(g, name, B)
        for k, v in prof.items():
            tr, lsu, src = ncu_for(k, B)
            stages[f"{op}:{k}"] = {"ms": v, "bytes": by[k], "GBps": by[k] / (v * 1e-3) / 1e9,
                                   "frac": by[k] / (v * 1e-3) / 1e9 / peak,
                                   "compulsory_bytes": comp[k],
                                   "frac_compulsory": comp[k] / (v * 1e-3) / 1e9 / peak,
                                   "traffic": tr, "traffic_over_bytes": (tr / by[k]) if tr else None,
                                   "l1_lsu_pct_ncu": lsu}
    total = sum(s["ms"] for s in stages.values())
    dom_name, dom = max(stages.items(), key=lambda kv: kv[1]["ms"])
    for s in stages.values():
        s["share"] = s["ms"] / total
    ncu_src = _ncu_capture()[1]

    # the reference's own sampling_plan (minimal N_rho, 4333 = 7 * 619 at
    # N=2048: its rho convolution runs zero-padded over 8748) on the same stack
    default_plan = None
    if args.plan == "smooth" and not args.no_default_plan:
        gd = geometry(args, "default")
        pd = lp.RadonPlan(gd, max_batch=B, device=local)
        hd = pd.handle
        sino_d = torch.empty(B, gd.n_theta, gd.N, device=dev)

        def step_d():
            lp._lib.check(L.lpr_gpu_radon(hd, imgs.data_ptr(), sino_d.data_ptr(), B, sp))
            lp._lib.check(L.lpr_gpu_backproject(hd, sino_d.data_ptr(), back.data_ptr(), B, sp))

        ms_d = timed(step_d, n=max(3, min(args.steps, 10)), warm=3)
        prof_d = roofline.profile_stages(pd, "radon", imgs.data_ptr(), sino_d.data_ptr(), B, 2)
        prof_db = roofline.profile_stages(pd, "backproject", sino_d.data_ptr(), back.data_ptr(), B, 2)
        default_plan = {"n_rho": gd.n_rho, "value": ws * B / (ms_d / 1e3), "unit": UNIT, "ms_per_step": ms_d,
                        "stages_ms": {**{f"R:{k}": v for k, v in prof_d.items()},
                                      **{f"R#:{k}": v for k, v in prof_db.items()}}}
        del sino_d
        pd.close()

    result = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            try:
                sec = cpu_sample(oracle_plan(args), z, zb)
                cpu = {"value": 1.0 / sec, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                       "sample": CPU_SAMPLE, "slices": 1}
            except Exception as e:  # the CPU leg is a reported baseline, not the product
                cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                       "sample": f"unavailable: {e}"}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config(args, g, ws),
            "radon_slices_per_s": ws * B / (ms_r / 1e3), "backproject_slices_per_s": ws * B / (ms_b / 1e3),
            "fbp_slices_per_s": ws * B / (ms_fbp / 1e3),
            "em_iterations": {"slice_iterations_per_s": ws * B / (ms_em / 1e3), "ms_per_iteration_per_slice": ms_em / B,
                              "how": "lpr_gpu_em, 3 iterations from f0 = 1 on the disc, clamped stack sinograms"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes_img,
                    "d2h_bytes_per_step": nbytes_sino + nbytes_img,
                    "how": "lpr_gpu_radon_backproject_host (R then R# in one call: images in, sinograms and "
                           "back-projections out) for steps 0..K-1, alternating between two host threads / plans; "
                           "pinned host buffers, every copy inside the wall clock, fill and drain included",
                    "pipelined_steps": e2e_pipe_k,
                    "link_bound_one_call_value": ws * B / ((nbytes_sino + nbytes_img) / (link["link_duplex_gbs"] * 1e9)),
                    "separate_calls": {"value": sep_value, "sequential_value": e2e_seq_value,
                                       "h2d_bytes_per_step": nbytes_img + nbytes_sino,
                                       "d2h_bytes_per_step": nbytes_sino + nbytes_img,
                                       "how": "lpr_gpu_radon_host of steps 0..K-1 on one host thread / plan and "
                                              "lpr_gpu_backproject_host of the same steps (each on its step's "
                                              "sinograms, re-uploaded) on a second, pipelined"},
                    **link},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": dom["GBps"], "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": dom["frac"],
                         "traffic": dom["traffic"], "share_of_step": dom["share"],
                         "l1_lsu_pct_ncu": dom["l1_lsu_pct_ncu"], "ncu_source": ncu_src,
                         "algorithmic_bytes_per_launch": dom["bytes"],
                         "bytes_model": "SURVEY.md §8(d) (fused kernels: sum of their stages)",
                         "frac_compulsory": dom["frac_compulsory"], "ms_per_launch": dom["ms"],
                         "step_frac": (roofline.slice_bytes(g, "radon") + roofline.slice_bytes(g, "backproject"))
                         * B / (ms_step * 1e-3) / 1e9 / peak},
            "stages": stages,
            "gathered": gathered,
            "stack": stack,
            "default_plan": default_plan,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(result), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    plan.close()
    return result


def run_dry(args):
    """--dry-run: the multi-rank plumbing of run_ours on CPU with gloo, no GPU
    and no measurement: world/--gpus check, slice sharding, max-over-ranks,
    and the final gather of every rank's (stand-in) sinograms to rank 0,
    verified element by element. Rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist

    from paper_1506_00014_b200 import sharding

    rank, ws, _ = world()
    if ws != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if ws > 1:
        dist.init_process_group("gloo")
    B, n_theta, N = args.batch, 3 * args.n // 2, args.n
    start, count = sharding.stack_shard(B * ws, ws, rank)
    sino = torch.arange(start, start + count, dtype=torch.float32).reshape(-1, 1, 1).expand(count, n_theta, N)
    sino = sino.contiguous()
    slowest = sharding.max_over_ranks(float(rank))
    out = sharding.gather_to_root(sino, 0)
    # the config-4 stack split: every slice of [0, stack) on exactly one rank
    s_start, s_count = sharding.stack_shard(args.stack, ws, rank)
    mine = torch.zeros(max(args.stack, 1), dtype=torch.int32)
    mine[s_start:s_start + s_count] = 1
    if ws > 1:
        dist.all_reduce(mine)
    stack_ok = bool((mine[:args.stack] == 1).all())
    line = None
    if rank == 0:
        ok = out is not None and out.shape[0] == B * ws and all(
            bool((out[i] == i).all()) for i in range(B * ws)) and stack_ok
        line = {"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": ws, "dry_run": True, "backend": "gloo",
                "config": {"N": N, "n_theta": n_theta, "global_batch": B * ws,
                           "parallelism": f"slices sharded dp{ws}"},
                "gathered": {"bytes_to_rank0_per_step": (ws - 1) * B * n_theta * N * 4, "verified": ok},
                "stack": {"slices": args.stack, "slices_per_rank0": s_count, "partition_verified": stack_ok},
                "max_over_ranks": slowest}
        print(json.dumps(line), flush=True)
        if not ok:
            raise SystemExit("dry run: gather mismatch")
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
