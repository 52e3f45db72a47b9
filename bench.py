"""Benchmark of the LOFP path sum on B200 (BASELINE.json metric: paths/s and amplitudes/s
on 1 B200; FP64-pipe fraction of roofline).

One *step* = one call of the hot path (``lofp_amplitudes``: Appendix-A tables when the
input changes, per-output column counts and unit split, the column-split enumeration,
the per-output reduction) over one batch of outputs resident in HBM.  The default
workload is BASELINE.json configs[4] (M=64, N=24, D=4) with its batch of 16384 outputs
conditioned on structural reachability and at most 1e9 paths per output (DESIGN.md
reading R14; the literal batch is ~100% structural zeros for configs[2] and 3e14 paths
per amplitude for configs[3]).  ``--config`` picks another config (0/1 literal batches,
2-4 conditioned), ``--literal`` the literal configs[4] batch (12,548 reachable outputs,
4.9e13 paths), ``--hero`` the 8 largest uncapped configs[4] outputs.  Inputs are the
seeded synthetic batches in data/ (written by scripts/make_batches.py).

Launch: ``python bench.py [--gpus N --steps K --warmup W]``; N > 1 under torchrun, one
rank per GPU, every rank evaluating the whole batch (weak scaling: per-GPU work fixed;
outputs are independent, so there is no collective on the data path).
``--impl reference`` times the CPU oracle instead.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DATA = os.path.join(ROOT, "data")
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["lofp", "reference"], default="lofp")
    p.add_argument("--config", type=int, default=4)
    p.add_argument("--outputs", type=int, default=0, help="limit the batch to its first N outputs")
    p.add_argument("--hero", action="store_true",
                   help="configs[4] hero sample: its 8 largest uncapped outputs (2.2e11-2.5e11 paths each)")
    p.add_argument("--literal", action="store_true",
                   help="configs[4] literal batch (reachable outputs only: 12,548 outputs, 4.9e13 paths)")
    p.add_argument("--contract", action="store_true",
                   help="time lofp_amplitudes_contract (strip tensor contraction, NEXT-1) instead of the path "
                        "sum; metric amplitudes/s (default workload then: configs[3] as literally drawn)")
    p.add_argument("--gates", action="store_true",
                   help="NEXT-3: add a Kerr phase gate exp(i(a n + b n^2)) on every mode after every layer "
                        "(P:338 'at essentially no additional cost')")
    p.add_argument("--nonlocal", dest="non_local", action="store_true",
                   help="NEXT-4: configs[4]'s mesh with long-range couplers (mode 4j+1 to 4j+4) in its second "
                        "layer instead of the nearest-neighbour pairs they displace; outputs = the conditioned batch")
    p.add_argument("--distribution", action="store_true",
                   help="NEXT-2: all C(N+M-1, M-1) outputs of configs[1]'s input in one call; metric amplitudes/s")
    p.add_argument("--tile", type=int, default=1,
                   help="--contract: the batch repeated this many times in one call (the 2048 outputs of "
                        "configs[3] are under one output per resident warp; copies fill the GPU)")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-paths", type=float, default=3e7, help="paths in the cpu_baseline sample")
    return p.parse_args()


def workload(idx: int, limit: int = 0, hero: bool = False, literal: bool = False):
    import lofp_inputs as li
    c = li.config(idx)
    d = np.load(os.path.join(DATA, f"cfg{idx}.npz"))
    if hero:  # uncapped single-output scaling sample (configs[4] only)
        T, P, kind = d["T_hero"].astype(np.int32), d["P_hero"].astype(np.uint64), "hero (uncapped)"
    elif literal:  # the literal batch, structural zeros dropped (they cost nothing)
        keep = d["P_literal"] > 0
        T, P = d["T_literal"][keep].astype(np.int32), d["P_literal"][keep].astype(np.uint64)
        kind = "literal (reachable rows)"
    elif "T_cond" in d.files:
        T, P, kind = d["T_cond"].astype(np.int32), d["P_cond"].astype(np.uint64), "conditioned"
    else:
        T, P, kind = d["T_literal"].astype(np.int32), d["P_literal"].astype(np.uint64), "literal"
    if limit:
        T, P = T[:limit], P[:limit]
    return c, T, P, kind


def aggregate(t_local_ms, paths_local, outs_local, world, dist=None, device=None):
    """Max of the ranks' device times, sums of their paths and outputs (the only
    collectives of the bench: there is none on the data path)."""
    import torch
    t = torch.tensor([t_local_ms], dtype=torch.float64, device=device)
    tot = torch.tensor([paths_local, outs_local], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    return float(t.item()), float(tot[0].item()), float(tot[1].item())


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    self.rows.append(parts)

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_sample(c, T, P, budget, seed=0):
    """A seeded random sample of the batch's outputs holding about `budget` paths (outputs
    larger than a quarter of the budget are skipped so the sample stays bounded)."""
    order = np.random.default_rng(seed).permutation(len(T))
    sel, tot = [], 0.0
    for i in order:
        p = float(P[i])
        if p > budget / 4:
            continue
        sel.append(int(i))
        tot += p
        if tot >= budget:
            break
    return np.sort(np.array(sel if sel else [int(np.argmin(P))], dtype=np.int64))


def run_oracle(c, T, P, sel, threads=0):
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    oracle.path_sum(c.M, c.layers, c.S, T[sel], threads=threads)
    dt = time.perf_counter() - t0
    return float(P[sel].astype(np.float64).sum()), dt


def reference_arm(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on the host cores, rank 0 only."""
    if rank != 0:
        return
    c, T, P, kind = workload(args.config, args.outputs)  # (no hero sample: hours on the CPU)
    sel = cpu_sample(c, T, P, args.cpu_paths / 4)
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        run_oracle(c, T, P, sel[: max(1, len(sel) // 8)])
    tot_paths, tot_s = 0.0, 0.0
    for _ in range(args.steps):
        p, dt = run_oracle(c, T, P, sel)
        tot_paths += p
        tot_s += dt
    v = tot_paths / tot_s
    line = {
        "impl": "reference", "metric": "paths/s", "value": v, "unit": "paths/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (long double accumulate)",
        "data": "synthetic", "config": {"workload": f"configs[{args.config}] {kind} batch (oracle sample)",
                                        "sample_outputs": int(len(sel))},
        "amplitudes_per_s": len(sel) * args.steps / tot_s,
        "cpu_baseline": {"value": v, "unit": "paths/s", "cores": cores, "kind": "oracle",
                         "sample": f"{len(sel)} outputs drawn at random from the batch (each <= 1/4 of the "
                                   f"path budget), {p:.3e} paths per step"},
        "e2e": {"value": v, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ncu_traffic(args):
    """DRAM bytes (read + write) per launch of the unit kernel from the committed ncu --set
    full capture of the same workload (profiles/r2_ncu_units_cfg<i>.txt), else None."""
    if args.hero or args.literal or args.outputs:
        return None
    path = os.path.join(ROOT, "profiles", f"r2_ncu_units_cfg{args.config}.txt")
    if not os.path.exists(path):
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for line in open(path):
        parts = line.split()
        if parts and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum") and len(parts) >= 3:
            tot += float(parts[1]) * scale.get(parts[2], 1)
    return {"bytes_per_launch": tot, "source": os.path.relpath(path, ROOT)} if tot else None


def nonlocal_layers(c):
    """configs[4]'s circuit with its second layer's pairs (4j+1, 4j+2), (4j+3, 4j+4) replaced
    by the long-range pairs (4j+1, 4j+4), (4j+2, 4j+3) (same angles): every fourth cut is
    crossed by a coupler spanning three cuts."""
    layers = [list(l) for l in c.layers]
    out = []
    l2 = {(a, b): (th, ph) for a, b, th, ph in layers[1]}
    done = set()
    for a, b, th, ph in layers[1]:
        j = (a - 1) // 4
        if (a - 1) % 4 == 0 and (a + 2, a + 3) in l2 and a not in done:
            th2, ph2 = l2[(a + 2, a + 3)]
            out.append((a, a + 3, th, ph))
            out.append((a + 1, a + 2, th2, ph2))
            done.update({a, a + 2})
        elif a not in done and (a - 3, a - 2) not in l2:
            out.append((a, b, th, ph))
    layers[1] = out
    return layers


def distribution_arm(args, rank, world, local):
    """--distribution: every output of configs[1]'s input (490,314 patterns) in one call."""
    import torch
    from paper_2510_26408_b200 import Circuit
    import lofp_inputs as li
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    c = li.config(1)
    circ = Circuit(c.M, c.layers)
    T, a = circ.distribution(c.S)
    torch.cuda.synchronize()
    tot = float(torch.sum(torch.abs(a) ** 2).item())
    if abs(tot - 1.0) > 1e-11:
        raise SystemExit(f"probabilities sum to {tot}")
    for _ in range(args.warmup):
        circ.distribution(c.S)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    ms = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        circ.distribution(c.S)
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    if rank == 0:
        B = len(T)
        line = {"metric": "amplitudes/s", "value": B * args.steps / (np.sum(ms) * 1e-3), "unit": "amplitudes/s",
                "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(ms)),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": f"configs[1] input, all {B} outputs (NEXT-2 lofp_distribution, contraction)",
                           "sum_p": tot}}
        print(json.dumps(line), flush=True)


def contract_roofline(terms, cmuls, kernel_ms):
    """Roofline of the contraction: FP64 lane instructions of its terms (a
    complex multiply-accumulate each, 4) and cut-factor products (4 per complex
    multiplication) over the call's device time, against the measured DFMA issue rate.  The
    kernel is issue/latency bound on the integer index work around those FP64 operations;
    the ncu capture of the same command (profiles/) gives its issue-slot utilisation."""
    from paper_2510_26408_b200 import _build
    lib = ctypes.CDLL(_build.PEAK_LIB)
    lib.lofp_probe_fp64_dfma_rate.restype = ctypes.c_double
    lib.lofp_probe_fp64_dfma_rate.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    nsm = ctypes.c_int(0)
    peak = lib.lofp_probe_fp64_dfma_rate(5, ctypes.byref(nsm)) / 1e12
    alg = 4.0 * terms + 4.0 * cmuls
    achieved = alg / (kernel_ms * 1e-3) / 1e12
    out = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFP64-inst/s",
           "frac": achieved / peak if peak > 0 else None, "traffic": None,
           "peak_source": f"measured DFMA issue rate (fp64_peak.cu, {nsm.value} SMs, burst)",
           "work_per_launch": {"terms": terms, "cmuls": cmuls, "fp64_lane_inst": alg},
           "kernel": "lofp_contract_warp_kernel", "kernel_ms": kernel_ms}
    prof = os.path.join(ROOT, "profiles", "r2_ncu_contract_warp_cfg3.txt")
    if os.path.exists(prof):
        for line in open(prof):
            if "smsp__issue_active.avg.pct_of_peak_sustained_active" in line:
                out["issue_active_ncu"] = float(line.split()[1]) / 100
            if line.startswith("  dram__bytes_read.sum") or line.startswith("  dram__bytes_write.sum"):
                v, u = float(line.split()[1]), line.split()[2]
                out["traffic"] = (out["traffic"] or 0) + v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        out["ncu_source"] = "profiles/r2_ncu_contract_warp_cfg3.txt"
    return out


def contract_arm(args, rank, world, local):
    """--contract: amplitudes/s of the strip tensor contraction on configs[3] as
    BASELINE.json draws it (2048 outputs, 2.5e18 paths: beyond any enumerator)."""
    import torch
    import torch.distributed as dist
    from paper_2510_26408_b200 import Circuit
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    idx = args.config if args.config != 4 else 3
    import lofp_inputs as li
    c = li.config(idx)
    d = np.load(os.path.join(DATA, f"cfg{idx}.npz"))
    T, P = d["T_literal"].astype(np.int32), d["P_literal"].astype(np.uint64)
    if args.outputs:
        T, P = T[:args.outputs], P[:args.outputs]
    if args.tile > 1:
        T, P = np.tile(T, (args.tile, 1)), np.tile(P, args.tile)
    B = len(T)
    circ = Circuit(c.M, c.layers)
    Td = torch.from_numpy(np.ascontiguousarray(T)).to(dev)
    out = torch.empty((B, 2), dtype=torch.float64, device=dev)
    counts = torch.zeros(B, dtype=torch.int64, device=dev)
    circ.contract(c.S, Td, out=out, counts=counts)
    torch.cuda.synchronize()
    vst = circ.stats()
    if not np.array_equal(counts.cpu().numpy().astype(np.uint64), P) or vst["unsupported"] or vst["check_errors"]:
        raise SystemExit("contraction path counts differ from the oracle's")
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        circ.contract(c.S, Td, out=out)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    clocks.start()
    ms = []
    for _ in range(args.steps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        circ.contract(c.S, Td, out=out)
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    clk = clocks.stop()
    t_max, paths_all, outs_all = aggregate(float(np.sum(ms)), float(P.astype(np.float64).sum()), float(B), world,
                                           dist, dev)
    value = outs_all * args.steps / (t_max * 1e-3)
    Th = torch.from_numpy(np.ascontiguousarray(T)).pin_memory()
    e2e = None
    if not args.no_e2e:
        # end to end: H2D of T and D2H of the amplitudes inside the timed region
        t0 = time.perf_counter()
        for _ in range(args.steps):
            Tg = Th.to(dev, non_blocking=True)
            a = circ.contract(c.S, Tg, out=out)
            a.cpu()
        dt = time.perf_counter() - t0
        e2e = {"value": B * args.steps / dt, "unit": "amplitudes/s", "h2d_bytes_per_step": int(T.nbytes),
               "d2h_bytes_per_step": int(B * 16)}
    if rank == 0:
        st = circ.stats()
        terms = int(st["terms"])
        line = {
            "metric": "amplitudes/s", "value": value, "unit": "amplitudes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"configs[{idx}] literal batch by the strip tensor contraction (NEXT-1): "
                                   f"M={c.M} N={c.N} D={c.D}, {B} outputs"
                                   + (f" (the batch x {args.tile})" if args.tile > 1 else "")
                                   + f", {float(P.astype(np.float64).sum()):.3e} "
                                   f"paths (not enumerated)", "global_batch": int(outs_all),
                       "l2": "flushed between steps (256 MiB write)"},
            "paths_equivalent_per_s": paths_all * args.steps / (t_max * 1e-3),
            "roofline": contract_roofline(terms, int(st["cmuls"]), float(np.mean(ms))),
            "e2e": e2e, "gpu_launches": int(st["launches"]) * args.steps, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2510_26408_b200 import Circuit
    from paper_2510_26408_b200 import _build

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    if args.contract:
        contract_arm(args, rank, world, local)
        return
    if args.distribution:
        distribution_arm(args, rank, world, local)
        return
    c, T, P, kind = workload(args.config, args.outputs, args.hero, args.literal)
    layers, gates = c.layers, []
    if args.gates:
        rng = np.random.default_rng(338)
        gates = [(m, l, float(rng.uniform(-3, 3)), float(rng.uniform(-1, 1)))
                 for l in range(c.D + 1) for m in range(c.M)]
        kind += f", {len(gates)} Kerr phase gates (NEXT-3)"
    if args.non_local:
        layers = nonlocal_layers(c)
        P = None
        kind += ", long-range couplers (NEXT-4)"
    circ = Circuit(c.M, layers, gates)
    Td = torch.from_numpy(np.ascontiguousarray(T)).to(dev)
    B = len(T)
    out = torch.empty((B, 2), dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    # validation pass (untimed): the path products the kernel formed per output must equal
    # the oracle's exact path counts (data/); its complex-multiplication count sizes the roofline
    counts = torch.zeros(B, dtype=torch.int64, device=dev)
    circ.amplitudes(c.S, Td, out=out, counts=counts)
    torch.cuda.synchronize()
    vst = circ.stats()
    got = counts.cpu().numpy().astype(np.uint64)
    if P is None:  # non-local workload: the oracle's counter is nearest-neighbour only; the kernel
        P = got    # checks its products against its own exact column count (check_errors)
    if not np.array_equal(got, P) or vst["check_errors"] or vst["unsupported"]:
        raise SystemExit(f"path counts differ from the oracle's on {int((got != P).sum())} outputs "
                         f"(check_errors={vst['check_errors']}, unsupported={vst['unsupported']})")
    cmuls, paths = int(vst["cmuls"]), int(vst["paths"])

    for _ in range(args.warmup):
        circ.amplitudes(c.S, Td, out=out)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ms, unit_ms = [], []
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush outside the timed events
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        circ.amplitudes(c.S, Td, out=out)
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        unit_ms.append(circ.stats()["units_ms"])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t_local = float(np.sum(ms))
    t_max, paths_all, outs_all = aggregate(t_local, float(P.astype(np.float64).sum()), float(B), world, dist, dev)
    value = paths_all * args.steps / (t_max * 1e-3)

    # end to end through the public host API: H2D of T, D2H of the amplitudes each step
    e2e = None
    if not args.no_e2e:
        Th = torch.from_numpy(np.ascontiguousarray(T)).pin_memory().numpy()
        circ.amplitudes_host(c.S, Th)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            circ.amplitudes_host(c.S, Th)
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": paths_all * args.steps / float(tt.item()), "unit": "paths/s",
               "h2d_bytes_per_step": int(T.nbytes), "d2h_bytes_per_step": int(B * 16)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel (the unit kernel): FP64 lane instructions the method
    # executes in this order = 4 per path (its product formed as a fused complex
    # multiply-accumulate: 2 DFMA per component) + 4 per other complex multiplication (the
    # half-path lists and their per-pair scalings: 2 DMUL + 2 DFMA), over the kernel's
    # device time (CUDA events on the launching stream, recorded inside liblofp)
    lib = ctypes.CDLL(_build.PEAK_LIB)
    lib.lofp_probe_fp64_dfma_rate.restype = ctypes.c_double
    lib.lofp_probe_fp64_dfma_rate.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    nsm = ctypes.c_int(0)
    peak_meas = lib.lofp_probe_fp64_dfma_rate(5, ctypes.byref(nsm)) / 1e12
    umean = float(np.mean(unit_ms))
    alg = 4.0 * paths + 4.0 * cmuls
    achieved = alg / (umean * 1e-3) / 1e12
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_meas, "unit": "TFP64-inst/s",
                "frac": achieved / peak_meas if peak_meas > 0 else None, "traffic": ncu_traffic(args),
                "peak_source": f"measured DFMA issue rate (fp64_peak.cu, {nsm.value} SMs, burst); "
                               f"MEASURED_PEAKS.json has no FP64 entry",
                "nominal_peak": 148 * 64 * 1965e6 / 1e12,
                "frac_of_nominal": achieved / (148 * 64 * 1965e6 / 1e12),
                "work_per_launch": {"paths": paths, "cmuls": cmuls, "fp64_lane_inst": alg},
                "kernel": "lofp_units_kernel", "kernel_ms": umean,
                "kernel_share_of_step": umean / (t_local / args.steps)}

    cpu = None
    if not args.no_cpu and world == 1 and not args.hero:  # (hero trees: hours on the CPU)
        sel = cpu_sample(c, T, P, args.cpu_paths)
        p, dt = run_oracle(c, T, P, sel)
        sel1 = cpu_sample(c, T, P, args.cpu_paths / 24, seed=1)
        p1, dt1 = run_oracle(c, T, P, sel1, threads=1)
        cpu = {"value": p / dt, "unit": "paths/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{len(sel)} outputs drawn at random from the batch ({p:.3e} paths), {dt:.1f} s",
               "one_core": {"value": p1 / dt1, "unit": "paths/s",
                            "sample": f"{len(sel1)} random outputs ({p1:.3e} paths), {dt1:.1f} s"}}

    line = {
        "metric": "paths/s", "value": value, "unit": "paths/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"configs[{args.config}] {kind} batch: M={c.M} N={c.N} D={c.D}, "
                               f"{B} outputs, {float(P.astype(np.float64).sum()):.4e} paths per GPU",
                   "global_batch": int(outs_all), "parallelism": f"the batch on each of {world} GPU(s)",
                   "l2": "flushed between steps (256 MiB write)"},
        "amplitudes_per_s": outs_all * args.steps / (t_max * 1e-3),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(vst["launches"]) * args.steps,  # this library's kernels per call
        "clocks": clk,
        "stats": {k: vst[k] for k in ("feasible", "units", "subsplits", "pairs", "elements", "max_list",
                                      "max_states", "table_entries", "grid_blocks", "block_threads")},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
