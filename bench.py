"""Benchmark: Steiner points inserted per second for gQM3D refinement.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gqm3d|reference]
                    [--config C4|C2|C5|C1|C3] [--scale S]

Workload (default C2, BASELINE configs[1]: the configuration the metric is
quoted on and the largest one the reference itself refines): 100,000 uniform
points + 1,000 random segments in the unit cube, B=1.6.  One step = one
complete refine of that PLC.  The north-star PLC C4 (outer icosphere r=1 +
inner icosphere r=0.45, level 6, 81,920 triangles each, + torus R=0.72 r=0.12,
40,000 triangles, + 1,000,000 points in the unit ball, B=1.5) is measured in
the same run under "north_star" (one refine capped at --north-star-rounds
rounds, the reference's own max_rounds knob) and selectable as the workload
with --config C4; C5 (the 64-PLC batch) with --config C5.

* value     Steiner/s with the PLC prepared and uploaded: GPU time of gq_refine
            (CUDA events on the context's stream, bulk Delaunay construction
            + every round + final verification), summed over the K steps
* e2e       Steiner/s through the public API refine(plc, cfg): host setup
            (validation incl. the device pair certifier, box closure, facet
            axes, insertion order), H2D, all rounds, D2H export of the mesh and
            the device quality report; wall clock per refine
* roofline  the Delaunay-region kernels (warp / block / huge tiers, SURVEY
            8(d): 58 B per tet tested + 24 B per candidate point) over their
            CUDA-event time, against the measured HBM copy peak; plus the
            whole-refine 8(d) byte formula over the whole device time
* cpu_baseline  the C++ oracle (sequential restatement of the reference, test
            infrastructure) on a bounded sample on this host, one core
Multi-GPU: refinement does not shard (BASELINE north_star): each rank refines
its own replica (C5: its share of the 64-PLC batch); no collectives on the
data path; value = all ranks' Steiner / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": (2.0, "unit cube + 1,000 uniform points (BASELINE configs[0])"),
    "C2": (1.6, "100,000 uniform points + 1,000 random segments in the unit cube (BASELINE configs[1])"),
    "C3": (1.4, "250,000 points + 2,000 axis-plane triangles on a 2^-16 grid (BASELINE configs[2], parity variant)"),
    "C4": (1.5, "nested icospheres (2 x 81,920 triangles) + torus (40,000 triangles) + 1,000,000 points in the "
                "unit ball (BASELINE configs[3], north-star target)"),
    "C5": (1.5, "batch of 64 unit cubes + 50,000 uniform points, seeds 0..63 (BASELINE configs[4])"),
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


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


def workload(config: str, scale: float = 1.0, rank: int = 0, world: int = 1):
    """The PLCs this rank refines in one step."""
    from paper_1903_03406_b200 import synth
    if config == "C5":
        n = max(1, int(64 * scale)) if scale < 1 else 64
        return [synth.cube_points(50000, seed) for seed in range(rank, n, world)]
    return [synth.config_plc(config, scale=scale)]


def cpu_sample(config: str, budget_s: float):
    """The oracle (C++ port of the reference, test infrastructure -- the only
    bench use of oracle/) on a bounded sample of the workload: the largest
    scale of the config whose refine fits the time budget, one core."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    from paper_1903_03406_b200 import synth
    B = CONFIGS[config][0]
    base = "C1" if config == "C5" else config
    scale = {"C1": 1.0, "C2": 0.1, "C3": 0.02, "C4": 0.0, "C5": 0.05}[config]
    if config == "C4":
        return None
    plc = synth.config_plc(base, scale=scale) if config != "C5" else synth.cube_points(int(50000 * scale), 0)
    t = time.perf_counter()
    out = oracle.refine(plc, B=B)
    dt = time.perf_counter() - t
    st = int((out["vert_origin"] == 1).sum())
    return {"value": st / dt, "unit": "steiner_points/s", "cores": 1, "kind": "port",
            "cpu": _cpu_model(), "cpus_on_host": os.cpu_count(),
            "sample": f"{config} scaled x{scale} ({len(plc.points)} points, {len(plc.segments)} segments, "
                      f"{len(plc.polygons)} polygons), full refine, {st} Steiner in {dt:.2f}s"}


def _oracle_run(config, scale, max_rounds, q):
    try:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle
        from paper_1903_03406_b200.prepare import prepare
        plcs = workload(config, scale)
        B = CONFIGS[config][0]
        st, tt, nr = 0, 0.0, 0
        for plc in plcs:
            prep = prepare(plc)
            t = time.perf_counter()
            out = oracle.refine_prepared(prep, B=B, max_rounds=max_rounds)
            tt += time.perf_counter() - t
            st += int((out["vert_origin"] == 1).sum())
            nr = max(nr, len(out.get("rounds", [])))
        q.put(("ok", st, tt, nr))
    except Exception as e:   # the reference's own behaviour on oblique facets
        q.put(("crashed", f"{type(e).__name__}: {str(e)[:200]}", 0.0, 0))


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (the C++ oracle port: the
    Python reference cannot travel to the GPU box) on the same config, one
    core per refine.  Each step is one full refine of the config's PLC (C5:
    the whole 64-PLC batch in a pool of host processes), under a wall cap;
    a configuration the port cannot finish is reported with its status."""
    if rank != 0:
        return
    import multiprocessing as mp
    B = CONFIGS[args.config][0]
    # C4: the port refines ~1 round per 100 s on this PLC and stops on oblique
    # facets later on, so both arms are compared at equal rounds
    max_rounds = args.ref_rounds if args.config == "C4" else args.max_rounds
    steps = max(1, min(args.steps, args.ref_steps if args.config != "C4" else 1))
    warm = 0
    times, steiner, status, rounds = [], [], "ok", 0
    for i in range(warm + steps):
        q = mp.get_context("fork").Queue()
        p = mp.get_context("fork").Process(target=_oracle_run, args=(args.config, args.scale, max_rounds, q))
        t0 = time.perf_counter()
        p.start()
        p.join(args.ref_cap_s)
        if p.is_alive():
            p.kill()
            p.join()
            status = f"did not finish within the {args.ref_cap_s:.0f} s cap"
            break
        res = q.get() if not q.empty() else ("crashed", "no result", 0.0, 0)
        if res[0] != "ok":
            status = f"crashed after {time.perf_counter() - t0:.1f} s: {res[1]}"
            break
        if i >= warm:
            steiner.append(res[1]); times.append(res[2]); rounds = res[3]
    value = sum(steiner) / sum(times) if times and sum(times) > 0 else None
    line = {"metric": "steiner_points_per_second", "value": value, "unit": "steiner_points/s", "n_gpus": world,
            "steps": len(times), "warmup": warm, "ms_per_step": 1000 * sum(times) / len(times) if times else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "status": status,
            "config": {"workload": f"{args.config}: {CONFIGS[args.config][1]}" + (f" scale {args.scale}" if args.scale != 1 else ""),
                       "B": B, "max_rounds": max_rounds, "rounds": rounds, "parallelism": "cpu-1core",
                       "same_config": True, "steps_requested": args.steps},
            "cpu_baseline": {"value": value, "unit": "steiner_points/s", "cores": 1, "kind": "port",
                             "cpu": _cpu_model(), "cpus_on_host": os.cpu_count(),
                             "sample": f"full {args.config} refine per step, {len(times)} step(s), "
                                       f"{sum(steiner)} Steiner in {sum(times):.1f} s" if times else status},
            "e2e": {"value": value, "unit": "steiner_points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def north_star(ctx, rounds: int, eq_rounds: int):
    """One C4 refine (the north-star PLC) with a round cap, device-timed, plus
    the same PLC stopped at the reference arm's equal-rounds cap."""
    from paper_1903_03406_b200.prepare import facet_keep, prepare
    from paper_1903_03406_b200 import synth
    B = CONFIGS["C4"][0]
    t0 = time.perf_counter()
    plc = synth.config_plc("C4")
    prep = prepare(plc, seed=0)
    keep = facet_keep(prep.plc)
    setup = time.perf_counter() - t0
    cnt = ctx.refine(prep, keep, B, rounds, 0)
    eq = ctx.refine(prep, keep, B, eq_rounds, 0)
    return {"workload": f"C4: {CONFIGS['C4'][1]}", "B": B, "max_rounds": rounds, "rounds": int(cnt.n_rounds),
            "steiner": int(cnt.steiner_points), "vertices": int(cnt.nv), "tet_slots": int(cnt.nt),
            "device_s": cnt.device_ms / 1000.0, "value": int(cnt.steiner_points) / (cnt.device_ms / 1000.0),
            "unit": "steiner_points/s", "host_setup_s": setup,
            "equal_rounds": {"rounds": int(eq.n_rounds), "steiner": int(eq.steiner_points),
                             "device_s": eq.device_ms / 1000.0,
                             "value": int(eq.steiner_points) / (eq.device_ms / 1000.0),
                             "reference_port": "34,960 Steiner in 190.8 s over the same 2 rounds on one core of the "
                                               "build container (183 Steiner/s; profiles/r02_summary.md)"},
            "skipped": int(cnt.n_skipped),
            "note": "one device-timed refine per bench run at the reference's default max_rounds (500): the "
                    "refine returns there like the reference's; it has not reached a fixed point yet "
                    "(faces still encroached, tet phase not started; DESIGN.md section 7)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gqm3d", choices=["gqm3d", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--north-star-rounds", type=int, default=500,
                    help="C2/C5 runs: also refine C4 once with this round cap (0: skip); "
                         "500 = the reference's default RefineConfig.max_rounds")
    ap.add_argument("--scale", type=float, default=1.0, help="workload scale (1.0 = the BASELINE config)")
    ap.add_argument("--max-rounds", type=int, default=500)
    ap.add_argument("--e2e-steps", type=int, default=3, help="end-to-end refines timed (<= --steps)")
    ap.add_argument("--ref-steps", type=int, default=2, help="reference arm: refines timed (<= --steps)")
    ap.add_argument("--ref-rounds", type=int, default=2,
                    help="C4: rounds both arms run for the like-for-like comparison (SURVEY 8(d): equal max_rounds; "
                         "the port needs ~100 s per C4 round)")
    ap.add_argument("--ref-cap-s", type=float, default=240.0, help="reference arm: wall cap per refine")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--streams", type=int, default=8, help="C5: PLCs in flight per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ["GQM3D_DEVICE"] = str(local)
    from paper_1903_03406_b200 import RefineConfig, refine
    from paper_1903_03406_b200 import _native
    from paper_1903_03406_b200.prepare import facet_keep, prepare

    B = CONFIGS[args.config][0]
    plcs = workload(args.config, args.scale, rank, world)
    cfg = RefineConfig(B=B, seed=0, max_rounds=args.max_rounds)
    preps = [prepare(p, seed=0) for p in plcs]
    keeps = [facet_keep(p.plc) for p in preps]
    ctx = _native.Context(local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    acc = {"steiner": 0, "dev_ms": 0.0, "region_ms": 0.0, "region_bytes": 0, "refine_bytes": 0, "launches": 0,
           "rounds": 0, "nt": 0, "nv": 0}

    concurrent = args.config == "C5"
    from paper_1903_03406_b200.replicas import refine_batch

    def device_step(record):
        if concurrent:   # the batch, args.streams PLCs in flight (one context + host thread each)
            cnts = refine_batch(plcs, cfg, local, args.streams, prepared=(preps, keeps))
        else:
            cnts = (ctx.refine(prep, keep, cfg.B, cfg.max_rounds, cfg.seed) for prep, keep in zip(preps, keeps))
        for cnt in cnts:
            if record:
                acc["steiner"] += int(cnt.steiner_points)
                acc["dev_ms"] += cnt.device_ms
                acc["region_ms"] += cnt.region_ms
                acc["region_bytes"] += int(cnt.bytes_alg)
                acc["refine_bytes"] += int(cnt.bytes_refine)
                acc["launches"] += int(cnt.kernel_launches)
                acc["rounds"] = int(cnt.n_rounds); acc["nt"] = int(cnt.n_real_tets or cnt.nt); acc["nv"] = int(cnt.nv)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        device_step(False)
    # ---- timed: device-resident path (inputs prepared and on the host once; each
    # refine uploads its few-MB PLC before the first event and builds everything on the device)
    batch_ms = 0.0
    with ClockSampler(local) as clk:
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            if concurrent:
                # several contexts' streams at once: device time of the whole batch,
                # CUDA events around it with the device drained on both sides
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                device_step(True)
                torch.cuda.synchronize()
                e1.record()
                e1.synchronize()
                batch_ms += e0.elapsed_time(e1)
            else:
                device_step(True)
        barrier()
        wall = time.perf_counter() - t0
    if concurrent:
        acc["dev_ms_sum"] = acc["dev_ms"]
        acc["dev_ms"] = batch_ms
    # ---- timed: end to end through the public API (host PLC in, mesh + report out).
    # refine() keeps its own per-device context: warm it once like the device arm.
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    if concurrent:
        refine_batch(plcs[:args.streams], cfg, local, args.streams)
    else:
        for p in plcs:
            refine(p, cfg)
    barrier()
    e0 = time.perf_counter()
    e2e_steiner = 0
    h2d = d2h = 0
    setup_s = 0.0
    for _ in range(e2e_steps):
        flush.zero_()
        outs = refine_batch(plcs, cfg, local, args.streams) if concurrent else (refine(p, cfg) for p in plcs)
        for mesh, rep in outs:
            e2e_steiner += rep.steiner_points
            setup_s += rep.device.get("prepare_s", 0.0)
    barrier()
    e2e_wall = time.perf_counter() - e0
    for prep in preps:
        h2d += prep.points.nbytes + prep.segments.nbytes + prep.poly_off.nbytes + prep.poly_idx.nbytes + prep.order.nbytes
    # bytes actually copied by gq_export_mesh (int32 ids on the wire) per PLC
    d2h = (mesh.nv * (24 + 1 + 4) + mesh.nt * (16 + 16 + 4 * 1 + 8)) * len(plcs)
    t_dev = acc["dev_ms"] / 1000.0
    tot_steiner = acc["steiner"]
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
        achieved = (acc["region_bytes"] / (acc["region_ms"] / 1000.0) / 1e9) if acc["region_ms"] > 0 else 0.0
        whole = acc["refine_bytes"] / (acc["dev_ms"] / 1000.0) / 1e9 if acc["dev_ms"] > 0 else 0.0
        try:   # the secondary roofline (FP64 predicate filters): measured FMA peak of this device
            fp64 = _native.probe_fp64(local)
        except Exception:
            fp64 = None
        traffic, traffic_note = None, None
        try:   # dram bytes of one captured region launch (ncu --set full), committed under profiles/
            with open(os.path.join(ROOT, "profiles", f"region_traffic_{args.config}.json")) as f:
                tr = json.load(f)
            traffic = tr["dram_bytes"]
            traffic_note = (f"{tr['kernel']} launch {tr['launch']} of a {args.config} refine: dram read+write "
                            f"{tr['dram_bytes']} B vs {tr['bytes_alg']} algorithmic B in {tr['duration_ms']} ms "
                            f"({tr['source']})")
        except Exception:
            pass
        n_plc = len(plcs) * world
        line = {
            "metric": "steiner_points_per_second", "value": tot_steiner / t_dev, "unit": "steiner_points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * t_dev / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {CONFIGS[args.config][1]}" + (f", scale {args.scale}" if args.scale != 1 else ""),
                       "B": B, "plcs_per_step": n_plc, "steiner_per_step": tot_steiner // args.steps,
                       "rounds": acc["rounds"], "vertices": acc["nv"], "tets": acc["nt"],
                       "parallelism": f"replicas x{world}" if args.config != "C5" else
                       f"PLC batch split over {world} GPU(s), {args.streams} PLCs in flight per GPU",
                       "l2": "flushed (256 MB write) before every step",
                       "refine_wall_s_per_step": wall / args.steps},
            "e2e": {"value": e2e_steiner / e2e_wall, "unit": "steiner_points/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "s_per_step": e2e_wall / e2e_steps, "steps": e2e_steps,
                    "host_setup_s_per_step": setup_s / e2e_steps},
            "gpu_launches": acc["launches"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic, "traffic_note": traffic_note,
                         "kernel": "Delaunay regions: k_region_warp / k_region_block / k_region_huge + bulk-construction "
                                   "k_init_region_warp (all launches, CUDA events)",
                         "whole_refine": {"achieved": whole, "frac": whole / peak if peak else None,
                                          "bytes_per_step": acc["refine_bytes"] // args.steps,
                                          "formula": "144 N_cand + 58 T_tested + 8 K_claims + 51 T_created + "
                                                     "1 T_deleted + 29 N_steiner (SURVEY 8(d))"},
                         "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)" if not peaks.get("_fallback") else "fallback",
                         "fp64_fma_peak_tflops": fp64},
            "clocks": clk.summary(),
        }
        if args.config == "C4":
            # like-for-like with the reference arm: the same PLC, the same round cap
            prep, keep = preps[0], keeps[0]
            cnt = ctx.refine(prep, keep, cfg.B, args.ref_rounds, cfg.seed)
            line["equal_rounds"] = {"rounds": int(cnt.n_rounds), "steiner": int(cnt.steiner_points),
                                    "device_s": cnt.device_ms / 1000.0,
                                    "value": int(cnt.steiner_points) / (cnt.device_ms / 1000.0),
                                    "note": "GPU refine stopped after the reference arm's round cap (--ref-rounds)"}
        if args.config != "C4" and args.north_star_rounds > 0 and world == 1:
            line["north_star"] = north_star(ctx, args.north_star_rounds, args.ref_rounds)
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_sample(args.config, args.cpu_budget_s)
            line["cpu_baseline"] = cb if cb else {
                "value": None, "unit": "steiner_points/s", "cores": 1, "kind": "port", "cpu": _cpu_model(),
                "sample": "none: the reference (and its port) cannot refine oblique facets (SURVEY F1); "
                          "see bench.py --impl reference for its status on this PLC"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
