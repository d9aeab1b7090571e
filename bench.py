"""Benchmark: Steiner points inserted per second for gQM3D refinement.

Workload (BASELINE.json configs[1]): 100k uniform points
+ 1k random segments in the unit cube, B=1.6, seed 0, one refine() per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gqm3d|reference]

* value     Steiner/s with the PLC already prepared and the mesh built on the
            device (sum of GPU event time of gq_refine over the K steps)
* e2e       Steiner/s through the public API refine(plc, cfg): host setup
            (validation, box closure, insertion order), H2D, all rounds,
            D2H export of the mesh and the quality report
* roofline  the Delaunay-region kernel (k_region), algorithmic bytes
            (58 B per tet tested + 24 B per candidate point)
            over its CUDA-event time, against the measured HBM copy peak
* cpu_baseline  the C++ oracle (sequential restatement of the reference) on a
            bounded sample on this host, one core
Multi-GPU: refinement does not shard (BASELINE north_star) -> N independent
replicas, one per rank, no collectives; value = all ranks' Steiner / max time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_C2 = 1.6


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 2 + k and r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def workload(scale: float = 1.0, seed: int = 0):
    from paper_1903_03406_b200 import synth
    return synth.config_plc("C2", scale=scale, seed=seed)


def cpu_baseline(sample_scale: float = 0.1):
    """The oracle (C++ port of the reference) on a bounded C2 sample, 1 core."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # test-infrastructure checker; the only bench use of oracle/
    plc = workload(sample_scale)
    t = time.perf_counter()
    out = oracle.refine(plc, B=B_C2)
    dt = time.perf_counter() - t
    st = int((out["vert_origin"] == 1).sum())
    return {"value": st / dt, "unit": "steiner_points/s", "cores": 1, "kind": "port",
            "sample": f"C2 scaled x{sample_scale} ({len(plc.points)} points, {len(plc.segments)} segments), "
                      f"full refine, {st} Steiner in {dt:.2f}s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    times, steiner = [], []
    for i in range(args.warmup + args.steps):
        res = cpu_baseline(args.ref_scale)
        if i >= args.warmup:
            st = int(res["sample"].split(", full refine, ")[1].split(" ")[0])
            times.append(st / res["value"])
            steiner.append(st)
    tot = sum(times)
    value = sum(steiner) / tot
    line = {"metric": "steiner_points_per_second", "value": value, "unit": "steiner_points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"C2 (100k pts + 1k segs, B=1.6) bounded sample: scale x{args.ref_scale}",
                       "B": B_C2, "parallelism": "cpu-1core"},
            "cpu_baseline": {"value": value, "unit": "steiner_points/s", "cores": 1, "kind": "port",
                             "sample": res["sample"]},
            "e2e": {"value": value, "unit": "steiner_points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gqm3d", choices=["gqm3d", "reference"])
    ap.add_argument("--scale", type=float, default=1.0, help="workload scale (1.0 = BASELINE C2)")
    ap.add_argument("--ref-scale", type=float, default=0.1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ["GQM3D_DEVICE"] = str(local)
    from paper_1903_03406_b200 import RefineConfig, refine
    from paper_1903_03406_b200 import _native
    from paper_1903_03406_b200.prepare import facet_keep, prepare

    plc = workload(args.scale)
    cfg = RefineConfig(B=B_C2, seed=0)
    prep = prepare(plc, seed=0)
    keep = facet_keep(prep.plc)
    ctx = _native.Context(local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def device_step():
        cnt = ctx.refine(prep, keep, cfg.B, cfg.max_rounds, cfg.seed)
        return cnt

    for _ in range(args.warmup):
        device_step()
    # ---- timed: device-resident path
    steiner = 0
    dev_ms = 0.0
    region_ms = 0.0
    region_bytes = 0
    launches = 0
    cnt = None

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            cnt = device_step()
            steiner += int(cnt.steiner_points)
            dev_ms += cnt.device_ms
            region_ms += cnt.region_ms
            region_bytes += int(cnt.bytes_alg)
            launches += int(cnt.kernel_launches)
        barrier()
        wall = time.perf_counter() - t0
    # ---- timed: end to end through the public API (host PLC in, mesh + report out).
    # refine() keeps its own per-device context: warm it up like the device arm
    # (first-call allocations are not part of a refine).
    for _ in range(args.warmup):
        refine(plc, cfg)
    barrier()
    e0 = time.perf_counter()
    e2e_steiner = 0
    for _ in range(args.steps):
        flush.zero_()
        mesh, rep = refine(plc, cfg)
        e2e_steiner += rep.steiner_points
    barrier()
    e2e_wall = time.perf_counter() - e0
    h2d = prep.points.nbytes + prep.segments.nbytes + prep.poly_off.nbytes + prep.poly_idx.nbytes + prep.order.nbytes
    d2h = (mesh.points.nbytes + mesh.vert_origin.nbytes + mesh.vert_tet.nbytes // 2 + mesh.tv.nbytes // 2
           + mesh.tn.nbytes // 2 + mesh.alive.nbytes + mesh.sub_mask.nbytes + mesh.seg_mask.nbytes
           + mesh.ratio.nbytes + mesh.skip_flag.nbytes)
    # max over ranks of the device time
    t_dev = dev_ms / 1000.0
    tot_steiner = steiner
    if world > 1:
        tt = torch.tensor([t_dev, e2e_wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev, e2e_wall = float(tt[0]), float(tt[1])
        ss = torch.tensor([tot_steiner, e2e_steiner], device="cuda", dtype=torch.float64)
        dist.all_reduce(ss)
        tot_steiner, e2e_steiner = int(ss[0]), int(ss[1])
    if rank == 0:
        peaks = _peaks()
        peak = float(peaks.get("hbm_gbs", 6650.0))
        achieved = (region_bytes / (region_ms / 1000.0) / 1e9) if region_ms > 0 else 0.0
        traffic, traffic_note = None, None
        try:   # dram bytes of one captured region launch (ncu --set full), committed under profiles/
            with open(os.path.join(ROOT, "profiles", "region_traffic.json")) as f:
                tr = json.load(f)
            traffic = tr["dram_bytes"]
            traffic_note = (f"{tr['kernel']} launch {tr['launch']} of a C2 refine: dram read+write {tr['dram_bytes']} B "
                            f"vs {tr['bytes_alg']} algorithmic B in {tr['duration_ms']} ms ({tr['source']})")
        except Exception:
            pass
        line = {
            "metric": "steiner_points_per_second", "value": tot_steiner / t_dev, "unit": "steiner_points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * t_dev / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C2: {len(plc.points)} points + {len(plc.segments)} segments in the unit cube, "
                                   f"B={B_C2}, seed 0 (BASELINE configs[1])", "steiner_per_step": steiner // args.steps,
                       "rounds": int(cnt.n_rounds), "tets": int(cnt.nt), "parallelism": f"replicas x{world}",
                       "l2": "flushed (256 MB write) before every step"},
            "wall_s_per_step": wall / args.steps,
            "e2e": {"value": e2e_steiner / e2e_wall, "unit": "steiner_points/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "s_per_refine": e2e_wall / args.steps},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic, "traffic_note": traffic_note,
                         "kernel": "k_region_warp + k_init_region_warp (Delaunay regions; all launches, CUDA events)",
                         "peak_source": "measured" if not peaks.get("_fallback") else "fallback"},
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(args.ref_scale)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
