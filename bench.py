#!/usr/bin/env python3
"""Throughput benchmark of the B200 list-CRC polar decoder.

One step = one decode of a batch of seeded BPSK-AWGN frames (the reference
harness's own per-frame generator) through the sm_100a kernel.  Default
workload: BASELINE.json's north star, (2048,1723) polar code with K including
CRC-32 (payload k = 1691), L = 32, float32, Eb/N0 = 4.0 dB.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3_L32]
  python bench.py --impl reference ...   # CPU oracle port on the host cores

Prints ONE JSON line (rank 0).  Multi-GPU: launched by torchrun, one rank per
GPU; each rank decodes its own frame shard (no data-path collective); the
only collective is the final NCCL all-reduce of timings and error counts.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import paper_1505_01466_b200 as pb  # noqa: E402

CONFIGS = {
    # name: (N, K incl. CRC, crc, design Eb/N0, L, Eb/N0, mode, label)
    "c1_L4": (1024, 512, "crc8_d5", 2.0, 4, 2.5, "f32", "c1"),
    "c2_L8": (1024, 860, "crc32", 4.0, 8, 4.0, "f32", "c2"),
    "c3_L1": (2048, 1723, "crc32", 4.0, 1, 4.0, "f32", "c3"),  # single-path pass (k_ssc)
    "c3_L2": (2048, 1723, "crc32", 4.0, 2, 4.0, "f32", "c3"),
    "c3_L8": (2048, 1723, "crc32", 4.0, 8, 4.0, "f32", "c3"),
    "c3_L32": (2048, 1723, "crc32", 4.0, 32, 4.0, "f32", "c3"),
    "c4_int8_L32": (2048, 1723, "crc32", 4.0, 32, 4.0, "int8", "c4"),
    "c5_L16": (8192, 6144, "crc32", 3.0, 16, 3.0, "f32", "c5"),
}
# adaptive decoding (reference AdaptiveDecoder listdec.py:437-459):
# the single-path pass first, the list only for CRC failures -- the decoder
# behind the paper's headline throughput table; not the north-star metric
for _base in ("c1_L4", "c2_L8", "c3_L8", "c3_L32", "c4_int8_L32", "c5_L16"):
    CONFIGS[_base + "_adaptive"] = CONFIGS[_base]
DEFAULT_CONFIG = "c3_L32"
METRIC = "decoded info Gbit/s, Fast-SSC list-CRC (2048,1723) L=32; FER parity vs oracle"


def crc_of(name):
    return {"crc8_d5": pb.CrcConfig(width=8, polynomial=0xD5), "crc32": pb.CRC32}[name]


def make_code(cfg_name):
    N, K, crc_name, design, L, ebn0, mode, label = CONFIGS[cfg_name]
    crc = crc_of(crc_name)
    k = K - crc.width
    spec = pb.CodeSpec.from_design_ebn0(N, k, crc, design)
    return spec, pb.build_schedule(spec), L, ebn0, mode, label


def lane_ops_per_frame(schedule, L):
    """W = L(3 S_F + 2 S_G + 2 S_R0 + 4 S_Rep + 4 S_R1 + 4 S_SPC)
    + sum over forking leaves of L*C (minimal 32-bit lane-instructions)."""
    S = dict(F=0, G=0, R0=0, REP=0, R1=0, SPC=0)
    fork = 0
    for op in schedule.ops:
        k = op.kind
        if k is pb.NodeKind.F:
            S["F"] += op.size // 2
        elif k is pb.NodeKind.G:
            S["G"] += op.size // 2
        elif k is pb.NodeKind.RATE0:
            S["R0"] += op.size
        elif k is pb.NodeKind.REP or (k is pb.NodeKind.RATE1 and op.size == 1):
            S["REP"] += op.size
            fork += 2
        elif k is pb.NodeKind.RATE1:
            S["R1"] += op.size
            fork += 4
        elif k is pb.NodeKind.SPC:
            S["SPC"] += op.size
            fork += 2 if L == 2 else 8
    return L * (3 * S["F"] + 2 * S["G"] + 2 * S["R0"] + 4 * S["REP"] + 4 * S["R1"]
                + 4 * S["SPC"]) + L * fork


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
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
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def parse_opts(items):
    """--opt key=value (repeatable) -> ListDecoder options (pb_options)."""
    out = {}
    for it in items or []:
        k, _, v = it.partition("=")
        out[k.strip()] = v.strip() if k.strip() == "kernel" else int(v)
    return out


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_rate(schedule, L, llrs, mode, seconds: float, adaptive: bool = False):
    """Info bits/s of the CPU oracle port on all host threads over a bounded
    sample (calibrated to ~`seconds` of work)."""
    from oracle import oracle
    threads = cpu_threads()
    int8 = mode == "int8"
    feed = pb.quantize_int8(llrs).astype(np.float32) if int8 else llrs
    run = oracle.adaptive_batch if adaptive else oracle.decode_batch
    probe = min(len(feed), max(threads, 2 * threads) * (16 if adaptive else 1))
    t0 = time.perf_counter()
    run(schedule, L, feed[:probe], int8=int8, threads=threads)
    dt = time.perf_counter() - t0
    n = int(min(len(feed), max(probe, probe * seconds / max(dt, 1e-6))))
    t0 = time.perf_counter()
    run(schedule, L, feed[:n], int8=int8, threads=threads)
    dt = time.perf_counter() - t0
    return n * schedule.spec.k / dt, n, threads, dt


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    spec, sch, L, ebn0, mode, label = make_code(args.config)
    threads = cpu_threads()
    # per-step sample: ~args.ref_step_s seconds of oracle work on all threads
    pool = pb.generate_frames(spec, ebn0, seed=args.seed, start=0,
                              count=max(4 * threads, 256))
    adaptive = args.config.endswith("_adaptive")
    rate, n, threads, _ = oracle_rate(sch, L, pool.llrs, mode, 2.0, adaptive)
    per_step = int(max(threads, min(len(pool.llrs) * 64, rate / spec.k * args.ref_step_s)))
    if per_step > len(pool.llrs):
        pool = pb.generate_frames(spec, ebn0, seed=args.seed, start=0, count=per_step)
    from oracle import oracle
    int8 = mode == "int8"
    feed = pb.quantize_int8(pool.llrs).astype(np.float32) if int8 else pool.llrs
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        (oracle.adaptive_batch if adaptive else oracle.decode_batch)(
            sch, L, feed[:per_step], int8=int8, threads=threads)
        if step >= args.warmup:
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = args.steps * per_step * spec.k / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gbit/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if mode == "f32" else "int8",
        "data": "synthetic (seeded BPSK-AWGN, reference per-frame Philox generator)",
        "config": config_dict(args, spec, L, ebn0, mode, label, args.batch),
        "cpu_baseline": {"value": value, "unit": "Gbit/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"each step decodes a bounded sample of the workload's "
                                   f"{args.batch}-frame batch: its first {per_step} frames "
                                   f"(x {args.steps} steps) through oracle/libpolar_oracle.so (C "
                                   f"restatement of polaris.listdec), {threads} threads"},
        "e2e": {"value": value, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def metric_of(cfg):
    if cfg.endswith("_adaptive"):
        return "decoded info Gbit/s, adaptive Fast-SSC + list-CRC (SSC pass, list on CRC failure)"
    return METRIC


def config_dict(args, spec, L, ebn0, mode, label, batch):
    dec = "adaptive (single-path pass, list on CRC failure), " if args.config.endswith("_adaptive") else ""
    return {"workload": f"{label}: polar ({spec.N},{spec.k_total}) incl. CRC-{spec.crc_width}"
                        f" (payload {spec.k}), {dec}L={L}, {mode}, Eb/N0={ebn0} dB",
            "config_key": args.config, "N": spec.N, "K": spec.k_total, "k_payload": spec.k,
            "list_size": L, "mode": mode, "ebn0_db": ebn0, "batch_frames": batch,
            "l2": "inputs larger than L2 (batch LLRs > 126 MB)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--seed", type=int, default=3040)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=6.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--opt", action="append", default=[],
                    help="decoder option key=value (pb_options: kernel, sync_every, ...)")
    ap.add_argument("--no-latency", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    spec, sch, L, ebn0, mode, label = make_code(args.config)
    B = args.batch
    # this rank's frame shard: frames [rank*B, (rank+1)*B) of the seeded stream
    frames = pb.generate_frames(spec, ebn0, seed=args.seed, start=rank * B, count=B)
    llr_host = torch.from_numpy(frames.llrs).pin_memory()
    llr_dev = llr_host.to(dev)
    info = torch.empty((B, spec.k), dtype=torch.uint8, device=dev)
    okd = torch.empty(B, dtype=torch.uint8, device=dev)
    pmd = torch.empty(B, dtype=torch.float64, device=dev)
    pud = torch.empty(B, dtype=torch.int32, device=dev)
    invd = torch.empty(B, dtype=torch.uint8, device=dev)
    adaptive = args.config.endswith("_adaptive")
    opts = parse_opts(args.opt)
    if adaptive:
        dec = pb.AdaptiveDecoder(sch, L, mode=mode, device=local, options=opts)
    else:
        dec = pb.ListDecoder(sch, L, mode=mode, device=local, options=opts)
    stream = torch.cuda.current_stream(dev)

    def step():
        if adaptive:
            dec.decode_device(llr_dev, info, okd, pmd, pud, invd)
        else:
            dec.decode_device(llr_dev, info, okd, pmd, pud)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = dec.launches
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clocks:
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    total_ms = evs[0].elapsed_time(evs[-1])
    launches = dec.launches - launches0

    # frame / bit errors of the last step vs the sent payloads (outside timing)
    pay = torch.from_numpy(frames.payloads).to(dev)
    bit_err = (info != pay).sum(dim=1)
    counters = torch.tensor([B, int((bit_err > 0).sum()), int(bit_err.sum())],
                            dtype=torch.float64, device=dev)
    tmax = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms = float(tmax.item())

    # end to end through the public API: pinned host LLRs in, host results out
    # (int8 mode: the fixed-point front end's int8 LLRs, a quarter of the bytes)
    if mode == "int8":
        llr_host = torch.from_numpy(pb.quantize_int8(frames.llrs)).pin_memory()
    in_bytes = B * spec.N * (1 if mode == "int8" else 4)
    info_h = torch.empty((B, spec.k), dtype=torch.uint8).pin_memory()
    ok_h = torch.empty(B, dtype=torch.uint8).pin_memory()
    pm_h = torch.empty(B, dtype=torch.float64).pin_memory()
    pu_h = torch.empty(B, dtype=torch.int32).pin_memory()
    out_h = (pb.AdaptiveBatchResult(info_h, ok_h, pm_h, pu_h, torch.empty(B, dtype=torch.uint8).pin_memory())
             if adaptive else pb.BatchResult(info_h, ok_h, pm_h, pu_h))
    e2e_steps = max(1, min(args.steps, 5))
    dec.decode_batch(llr_host, out=out_h)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dec.decode_batch(llr_host, out=out_h)
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_t.item())

    # single-frame latency (the paper's per-frame figure):
    # one frame per launch, device-resident (CUDA events) and through decode()
    latency = None
    if rank == 0 and not args.no_latency:
        one = llr_dev[:1].contiguous()
        lat_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        dev_us, api_us = [], []
        for i in range(60):
            lat_ev[0].record(stream)
            if adaptive:
                dec.decode_device(one, info[:1], okd[:1], pmd[:1], pud[:1], invd[:1])
            else:
                dec.decode_device(one, info[:1], okd[:1], pmd[:1], pud[:1])
            lat_ev[1].record(stream)
            torch.cuda.synchronize(dev)
            if i >= 10:
                dev_us.append(1e3 * lat_ev[0].elapsed_time(lat_ev[1]))
        host_one = frames.llrs[0] if mode == "f32" else pb.quantize_int8(frames.llrs[:1])[0]
        for i in range(30):
            t0 = time.perf_counter()
            dec.decode(host_one)
            if i >= 5:
                api_us.append(1e6 * (time.perf_counter() - t0))
        latency = {"frame_p50_us_device": statistics.median(dev_us),
                   "frame_p50_us_e2e": statistics.median(api_us),
                   "note": "one frame per launch; device: CUDA events around the decode kernel(s); "
                           "e2e: ListDecoder.decode(llr) wall time incl. copies and launch"}

    if rank == 0:
        frames_all = B * world
        value = frames_all * args.steps * spec.k / (total_ms * 1e-3) / 1e9
        peaks, peak_kind = load_peaks()
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        W = lane_ops_per_frame(sch, L)
        inv_frac = float(invd.float().mean()) if adaptive else 1.0
        if adaptive:  # single-path work for every frame + list work for the invoked ones
            W = lane_ops_per_frame(sch, 1) + inv_frac * W
        kernel_ms = (total_ms / max(1, launches) if world == 1 and not adaptive
                     else total_ms / args.steps)
        achieved = W * B / (kernel_ms * 1e-3) / 1e9           # G lane-ops/s, one GPU
        peak = sms * 128 * sm_mhz * 1e6 / 1e9
        hbm_bytes = B * (spec.N * 4 + spec.k + 13)
        hbm_gbs = hbm_bytes / (kernel_ms * 1e-3) / 1e9
        # measured DRAM traffic of the decode kernel: dram__bytes_read + dram__bytes_write of one
        # `ncu --set full` capture of this config (profiles/ncu_<config>.json, tools/ncu_summary.py),
        # per frame, times the frames of one launch
        traffic = traffic_frames = None
        prof = os.path.join(REPO, "profiles", f"ncu_{args.config}.json")
        if os.path.exists(prof):
            try:
                with open(prof) as fh:
                    pj = json.load(fh)
                traffic = pj.get("dram_bytes_per_launch_per_frame")
                traffic_frames = pj.get("frames")
                traffic = None if traffic is None else traffic * B
            except Exception:
                traffic = None
        line = {
            "metric": metric_of(args.config), "value": value, "unit": "Gbit/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if mode == "f32" else "int8",
            "data": "synthetic (seeded BPSK-AWGN frames from the reference's per-frame Philox "
                    "generator; random payloads)",
            "config": config_dict(args, spec, L, ebn0, mode, label, B),
            "p50_batch_ms": statistics.median(step_ms),
            "frames_per_s": frames_all * args.steps / (total_ms * 1e-3),
            "fer": float(counters[1] / counters[0]), "ber": float(counters[2] / (counters[0] * spec.k)),
            "gpu_launches": int(launches),
            "e2e": {"value": frames_all * e2e_steps * spec.k / e2e_s / 1e9, "unit": "Gbit/s",
                    "h2d_bytes_per_step": in_bytes,
                    "d2h_bytes_per_step": B * (spec.k + 1 + 8 + 4 + (1 if adaptive else 0))},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Glane-op/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "work_per_frame_lane_ops": W,
                         "peak_note": f"{sms} SMs x 128 lanes x {sm_mhz:.0f} MHz "
                                      f"(sm_max_mhz, {peak_kind}); SURVEY 8(d) ALU-issue roofline",
                         "hbm_gbs": hbm_gbs, "hbm_frac": hbm_gbs / float(peaks.get("hbm_gbs", 6650.0)),
                         # the same from the measured DRAM bytes (global alpha scratch included)
                         "dram_gbs_measured": None if traffic is None else traffic / (kernel_ms * 1e-3) / 1e9,
                         "dram_frac_measured": None if traffic is None else
                         traffic / (kernel_ms * 1e-3) / 1e9 / float(peaks.get("hbm_gbs", 6650.0)),
                         "traffic_capture_frames": traffic_frames},
            "clocks": clocks.summary(),
            "latency": latency,
            "options": opts,
            "plan": json.loads((dec._list if adaptive else dec).plan),
        }
        if not args.no_cpu_baseline:
            rate, n, threads, dt = oracle_rate(sch, L, frames.llrs, mode, args.cpu_seconds, adaptive)
            line["cpu_baseline"] = {"value": rate / 1e9, "unit": "Gbit/s", "cores": threads,
                                    "kind": "port", "cpu_model": cpu_model(),
                                    "sample": f"{n} frames of the same batch through "
                                              f"oracle/libpolar_oracle.so ({dt:.1f} s, "
                                              f"{threads} threads)"}
        if adaptive:
            line["list_invoked_frac"] = inv_frac
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
