#!/usr/bin/env python
"""bench.py — time-to-fixpoint and join tuples/sec of the B200 GDlog hot path.

Contract (driver): `python bench.py --gpus N --steps K --warmup W [--impl ours|reference]`.
A "step" is one complete semi-naive evaluation (load EDB -> seed -> iterate to
the fixpoint) of the benchmark workload: BASELINE.json configs[1], transitive
closure on a synthetic power-law DAG of ~5M edge draws (workload c2_tc_pl,
paper_2311_02206_b200/workloads.py).  `value` = join tuples produced per
second of device time with the EDB already resident in HBM; `e2e` = the same
metric through the C-ABI with host buffers (EDB upload + output-relation
download inside the timed region).  N > 1 runs the hash-partitioned engine
(one rank per GPU, NCCL all-to-all per iteration) on the same graph.

Rank 0 prints ONE JSON line.  `--impl reference` times the reference CPU
engine (oracle/_ref, compiled from the unmodified arraylog headers) on the
box's host cores over a bounded sample of the same generator.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# C2 workload (calibrated on B200 so |Reach| lands near 1e9)
C2 = dict(n=5_000_000, m=5_000_000, window=200, alpha=1.05, seed=1)
# bounded CPU sample of the same generator (reference engine ~10-30 s on 16 cores)
CPU_SAMPLE = dict(n=200_000, m=200_000, window=200, alpha=1.05, seed=1)
# The reference engine on the full C2 input is not attempted: SURVEY §8d
# extrapolates hours of CPU time, and its row-major u64 relations
# (|Reach| 7.7e8 rows x 16 B, plus the merge buffer and copies) exceed the
# host RAM of the survey box (62 GB).
FULL_SCALE_DNF = ("full C2 (n=m=5e6, |Reach|=7.7e8) not run on the CPU: DNF by SURVEY §8d's extrapolation "
                  "(hours; > 62 GB of host RAM for the u64 relation, its merge buffer and copies)")
PROGRAM = "reach"
HEAD = "Reach"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_rank{device}.csv"

    def start(self):
        if os.environ.get("GD_BENCH_CLOCK_MS") == "0":  # diagnostics only: no sampling
            return
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.f = open(self.path, "w")
            ms = os.environ.get("GD_BENCH_CLOCK_MS", "200")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", ms],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def flush_l2(torch, buf):
    mode = os.environ.get("GD_BENCH_FLUSH", "add")  # diagnostics: add | fill | none | addsleep
    if mode == "none":
        return
    if mode == "fill":
        buf.fill_(1)  # 256 MiB write > 126 MB L2
        return
    buf.add_(1)  # 256 MiB read-modify-write > 126 MB L2
    if mode == "addsleep":
        torch.cuda.synchronize()
        time.sleep(0.02)


def gen_workload():
    from paper_2311_02206_b200 import workloads as W
    return W.tc_pl(C2["n"], C2["m"], C2["window"], C2["alpha"], C2["seed"])


# ---------------------------------------------------------------------------

def cpu_baseline_sample():
    """The reference engine timed on a bounded sample (rank 0, N=1)."""
    from oracle.bindings import RefOracle
    from paper_2311_02206_b200 import abi as A
    from paper_2311_02206_b200 import workloads as W

    s = CPU_SAMPLE
    edges = W.tc_pl(s["n"], s["m"], s["window"], s["alpha"], s["seed"])
    ref = RefOracle()
    cfg = A.gd_engine_config((1 << 64) - 1, 1, 5, 0.8, 0, 0, 0)
    e = ref.engine(PROGRAM, cfg)
    t0 = time.perf_counter()
    e.load_edb("Edge", edges)
    e.run()
    dt = time.perf_counter() - t0
    return e, edges, dt


def join_tuples_of(edges: np.ndarray, reach: np.ndarray) -> int:
    """J summed over all iterations for Reach(f,t) :- Edge(f,m), Reach(m,t):
    every Reach row enters Δ exactly once and joins with indeg(m) edges, so
    ΣJ = Σ_{(m,t) in Reach} indeg(m) (indeg over distinct edges)."""
    e = np.unique(edges, axis=0)
    indeg = np.bincount(e[:, 1].astype(np.int64), minlength=int(max(e.max(), reach.max() if len(reach) else 0)) + 1)
    return int(indeg[reach[:, 0].astype(np.int64)].sum())


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(n: int) -> int:
    """Re-runs this command as N ranks (one per GPU) under torchrun; NCCL
    prints its communicator init lines (nRanks) to stderr."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    log("bench: launching", " ".join(cmd[2:]))
    return subprocess.call(cmd, env=env)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="diagnostics: run the multi-GPU (hash-partitioned, NCCL) path even at one rank")
    args = ap.parse_args()

    if args.impl == "reference":
        run_reference_main(args)
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: one rank per GPU under torchrun
        sys.exit(relaunch(args.gpus))

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    part = world > 1 or args.partitioned
    if part:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        log(f"rank {rank}: NCCL process group up, nranks {world}, device cuda:{local}")

    from paper_2311_02206_b200 import arraylog as al
    from paper_2311_02206_b200.partition import NcclComm, TorchExchange, run_partitioned

    # the engine runs on this (non-default) stream and every timing event is
    # recorded on it, so device times include all the engine's queued work
    # (the legacy default stream would be handed over as "no stream" and
    # the context would create its own)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = al.Context(local, stream.cuda_stream)
    assert stream.cuda_stream != 0, "the engine needs a real stream to be timed on"
    edges = gen_workload()
    d_edges = torch.from_numpy(edges.view(np.int64)).cuda()
    flush = torch.empty(256 << 20 >> 2, dtype=torch.int32, device="cuda")
    # N > 1: the library's native driver (its own NCCL send/recv on the
    # engine stream, one readback per iteration); GD_PART_DRIVER=python
    # runs the torch.distributed protocol (partition.run_partitioned)
    native = part and os.environ.get("GD_PART_DRIVER", "native") != "python"
    exch = TorchExchange() if part and not native else None
    comm = NcclComm(ctx, rank, world) if native else None

    def drive(e):
        if native:
            e.run_partitioned(comm)
        else:
            run_partitioned(e, exch, world)

    def one_step():
        e = al.engine(PROGRAM, ctx=ctx)
        if part:
            e.set_partition(rank, world)
        e.load_edb_device("Edge", d_edges.data_ptr(), len(edges))
        if part:
            e.seed()
            drive(e)
        else:
            e.run()
        return e

    # warm-up (also the parity/size record)
    for i in range(args.warmup):
        e = one_step()
        if i == 0:
            reach_n = e.relation_count(HEAD)
            iters = e.raw_stats().iterations
            jt = e.raw_stats().join_tuples
            log(f"warmup: |Edge|={len(edges)} |{HEAD}|={reach_n} iterations={iters} J={jt}")
        e.close()
        torch.cuda.synchronize()

    # timed steps (no per-kernel events inside: they would perturb the step)
    sampler = ClockSampler(local)
    launches0 = ctx.kernel_launches
    times, joins = [], []
    step_detail = []
    canary = torch.empty(21 << 27, dtype=torch.int64, device="cuda") if os.environ.get("GD_BENCH_CANARY") else None
    canary_ms = []
    hc0 = ctx.host_counters()
    sampler.start()
    for _ in range(args.steps):
        flush_l2(torch, flush)
        if part:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        e = one_step()
        t1.record(stream)
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        ph = e.stats().phase_seconds
        hc = ctx.host_counters()
        step_detail.append({k: round(v * 1e3, 1) for k, v in ph.items()} |
                           {"alloc_ms": round((hc["alloc_s"] - hc0["alloc_s"]) * 1e3, 1),
                            "allocs": hc["allocs"] - hc0["allocs"]})
        hc0 = hc
        jt = e.raw_stats().join_tuples
        reach_n = local_n = e.relation_count(HEAD)
        iters = e.raw_stats().iterations
        if part:
            mx = torch.tensor([ms], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
            sm = torch.tensor([jt, reach_n], dtype=torch.int64, device="cuda")
            torch.distributed.all_reduce(sm)
            ms, jt, reach_n = float(mx.item()), int(sm[0].item()), int(sm[1].item())
        times.append(ms)
        joins.append(jt)
        if _ == args.steps - 1:  # parity of the measured run (outside the timed region)
            digest = e.relation_digest(HEAD)
            if part:
                dg = torch.tensor([digest - (1 << 63)], dtype=torch.int64, device="cuda")
                dl = [torch.zeros_like(dg) for _ in range(world)]
                torch.distributed.all_gather(dl, dg)
                digest = sum(int(x.item()) + (1 << 63) for x in dl) % (1 << 64)
            step_record = {"count": int(reach_n), "digest": f"{digest:016x}", "iterations": int(iters),
                           "join_tuples": int(jt)}
        e.close()
        if canary is not None:  # diagnostics: GPU memory-op speed outside the engine
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            canary.fill_(-1)
            c1.record(stream)
            torch.cuda.synchronize()
            canary_ms.append(round(c0.elapsed_time(c1), 1))
    clocks = sampler.stop()
    launches = ctx.kernel_launches - launches0

    # one more identical step with CUDA events around every instrumented
    # launch (on the launching stream): per-kernel durations and their
    # algorithmic bytes for the roofline
    prof, prof_ms = {}, None
    if not args.no_profile:
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        ctx.set_profiling(True)
        ctx.profile_reset()
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        e = one_step()
        p1.record(stream)
        torch.cuda.synchronize()
        prof_ms = p0.elapsed_time(p1)
        prof = ctx.profile()
        ctx.set_profiling(False)
        e.close()

    ms_step = float(np.mean(times))
    value = float(np.mean(joins)) / (ms_step / 1e3)

    # roofline of the dominant kernel class
    peak, peak_kind = measured_peaks()
    roof = None
    if prof:
        dom = max(prof, key=lambda k: prof[k][0])
        ms_k, n_k, by_k = prof[dom]
        achieved = (by_k / n_k) / (ms_k / n_k / 1e3) / 1e9 if n_k and ms_k else 0.0
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_kind, "traffic": None,
                "launches": n_k, "avg_launch_ms": ms_k / max(n_k, 1),
                "algo_bytes_per_launch": by_k / max(n_k, 1),
                "share_of_step": ms_k / prof_ms, "profiled_step_ms": prof_ms}
        tp = ROOT / "profiles" / "ncu_traffic.json"
        if tp.exists():
            d = json.loads(tp.read_text()).get(dom)
            if d:
                roof["traffic"] = d.get("dram_bytes")
                roof["traffic_algo_bytes"] = d.get("algo_bytes")
                roof["traffic_source"] = d.get("source")
        # The fused insert is bound by random 8-byte slot CASes, each of which
        # moves a ~111-byte line of DRAM traffic on B200: report its measured
        # DRAM traffic (ncu) against the measured random-CAS ceiling too.
        rc = ROOT / "profiles" / "random_access_ceiling.json"
        if dom == "join_insert" and roof.get("traffic") and rc.exists():
            ceil = json.loads(rc.read_text())
            gbs = roof["traffic"] / (roof["avg_launch_ms"] / 1e3) / 1e9
            roof["random_access"] = {"dram_gbs": gbs, "ceiling_gbs": ceil["cas_dram_tbps"] * 1e3,
                                     "frac": gbs / (ceil["cas_dram_tbps"] * 1e3), "ceiling_source": ceil["source"]}
        # op-rate view of the fused insert: join rows settled per second of
        # insert-kernel time against the measured random 8-byte access
        # ceilings of this B200 (every join row is one random slot access)
        if dom == "join_insert" and rc.exists():
            ceil = json.loads(rc.read_text())
            ins_ms = prof["join_insert"][0]
            rate = float(np.mean(joins)) / (ins_ms / 1e3) / 1e9 if ins_ms else 0.0
            roof["op_rate"] = {"achieved_gops": rate, "unit": "G join rows/s",
                               "ceiling_load_gops": ceil["load_gops"], "ceiling_cas_gops": ceil["cas_gops"],
                               "frac_of_load_ceiling": rate / ceil["load_gops"],
                               "frac_of_cas_ceiling": rate / ceil["cas_gops"], "ceiling_source": ceil["source"]}
        jm = [k for k in ("join_probe", "join_materialize", "join_insert", "diff_merge", "difference")]
        jm_ms = sum(prof[k][0] for k in jm)
        jm_by = sum(prof[k][2] for k in jm)
        roof["join_merge"] = {"achieved": jm_by / (jm_ms / 1e3) / 1e9 if jm_ms else 0.0,
                              "frac": (jm_by / (jm_ms / 1e3) / 1e9) / peak if jm_ms else 0.0}
        roof["kernel_ms_per_step"] = {k: round(v[0], 3) for k, v in prof.items()}
        roof["kernel_gbs"] = {k: round(v[2] / (v[0] / 1e3) / 1e9, 1) for k, v in prof.items() if v[0] and v[2]}

    # e2e through the C-ABI with host buffers: every rank uploads the EDB
    # from pinned host memory, runs (partitioned at N > 1) and downloads
    # its shard of the result into pinned host rows; max over ranks
    e2e = None
    if not args.no_e2e:
        host_edges = torch.from_numpy(edges.view(np.int64)).pin_memory().numpy().view(np.uint64)
        out = torch.empty((max(local_n, 1), 2), dtype=torch.int64).pin_memory().numpy().view(np.uint64)
        e2e_t, e2e_parts = [], []
        h0 = d0 = 0
        # one untimed warm-up pass first (like the device steps' warm-up: the
        # download path's first call pays one-time host/device allocations)
        n_e2e = max(1, min(args.steps, 3))
        for it_e2e in range(n_e2e + 1):
            if it_e2e == 1:
                e2e_t, e2e_parts = [], []
                h0, d0 = ctx.transfer_bytes()
            if part:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e = al.engine(PROGRAM, ctx=ctx)
            if part:
                e.set_partition(rank, world)
            e.load_edb("Edge", al.tuple_array(2, host_edges))
            t1 = time.perf_counter()
            if part:
                e.seed()
                drive(e)
            else:
                e.run()
            n = e.relation_count(HEAD)
            t2 = time.perf_counter()
            ctx.check(ctx.lib.gd_engine_relation_download(e.h, 1, out.ctypes.data, n))
            dt = time.perf_counter() - t0
            e2e_parts.append((round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1), round((dt - (t2 - t0)) * 1e3, 1)))
            e.close()
            if part:
                mx = torch.tensor([dt], dtype=torch.float64, device="cuda")
                torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
                dt = float(mx.item())
            e2e_t.append(dt)
        h1, d1 = ctx.transfer_bytes()
        k = len(e2e_t)
        hb, db = (h1 - h0) // k, (d1 - d0) // k
        if part:  # whole-job bytes: sum over ranks
            sb = torch.tensor([hb, db], dtype=torch.int64, device="cuda")
            torch.distributed.all_reduce(sb)
            hb, db = int(sb[0].item()), int(sb[1].item())
        # bytes that crossed PCIe (the C-ABI counts every copy); the Reach
        # download moves 32-key blocks of byte-aligned offsets, rebuilt into
        # the caller's u64 rows by host threads (DESIGN.md §7 download)
        e2e = {"value": float(np.mean(joins)) / float(np.mean(e2e_t)), "unit": "tuples/s",
               "h2d_bytes_per_step": int(hb), "d2h_bytes_per_step": int(db),
               "host_rows_bytes": int(reach_n * 16), "seconds_per_step": float(np.mean(e2e_t)),
               "step_s": [round(t, 4) for t in e2e_t],
               "step_parts_ms": [{"load": a, "run": b, "download": c} for a, b, c in e2e_parts]}

    # parity of the measured C2 run: the committed full-scale record
    # (tests/golden/scale_digests.json: resident loop == host loop ==
    # partitioned P = 2/4/8, rows canonical, Σ Δ = |F|, ΣJ = Σ indeg)
    parity = {"c2_record": step_record}
    gp = ROOT / "tests" / "golden" / "scale_digests.json"
    if gp.exists():
        g = json.loads(gp.read_text()).get("c2_tc_pl")
        if g:
            want = {k: g["record"][k] for k in step_record}
            parity["c2_matches_golden"] = step_record == want

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            e, cedges, dt = cpu_baseline_sample()
            r = e.relation(HEAD)
            cj = join_tuples_of(cedges, r)
            # the same sample through the device path: byte-identical rows,
            # identical Δ history and join tuple count
            g = al.engine(PROGRAM, ctx=ctx)
            g.load_edb("Edge", al.tuple_array(2, cedges))
            g.run()
            parity["cpu_sample_bit_exact"] = bool(np.array_equal(g.relation(HEAD).data, r)
                                                  and g.delta_history(HEAD) == e.delta_history(HEAD)
                                                  and g.raw_stats().join_tuples == cj)
            g.close()
            s = CPU_SAMPLE
            cpu = {"value": cj / dt, "unit": "tuples/s", "cores": os.cpu_count(), "kind": "reference",
                   "cpu_model": cpu_model(), "threads": "engine_config.workers = 0 (all host threads)",
                   "sample": f"tc_pl n={s['n']} m={s['m']} W={s['window']} alpha={s['alpha']}: "
                             f"|Reach|={len(r)} J={cj} in {dt:.2f}s",
                   "time_to_fixpoint_s": dt, "full_scale": FULL_SCALE_DNF}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "error": str(ex)[:200]}

    if rank == 0:
        line = {
            "metric": "join_tuples_per_sec", "value": value, "unit": "tuples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "time_to_fixpoint_s": ms_step / 1e3,
            "config": {"workload": "c2_tc_pl", "program": PROGRAM, **C2, "edges": int(len(edges)),
                       "reach": int(reach_n), "iterations": int(iters), "join_tuples": int(np.mean(joins)),
                       "parallelism": (f"hash-partitioned x{world}" + (" (native NCCL driver)" if native else
                                                                         " (torch.distributed driver)"))
                       if part else "single",
                       "l2": "flushed between steps (256 MiB write)"},
            "step_ms": [round(t, 2) for t in times], "step_phases_ms": step_detail,
            **({"canary_fill_ms": canary_ms} if canary_ms else {}),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "parity": parity,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if part:
        torch.distributed.destroy_process_group()


def run_reference_main(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    times, joins = [], []
    for i in range(args.warmup + args.steps):
        e, edges, dt = cpu_baseline_sample()
        r = e.relation(HEAD)
        j = join_tuples_of(edges, r)
        log(f"reference step {i}: {dt:.2f}s |Reach|={len(r)} iters={e.stats().iterations} J={j}")
        if i >= args.warmup:
            times.append(dt)
            joins.append(j)
    t = float(np.mean(times))
    v = float(np.mean(joins)) / t
    s = CPU_SAMPLE
    line = {
        "impl": "reference", "metric": "join_tuples_per_sec", "value": v, "unit": "tuples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "time_to_fixpoint_s": t,
        "config": {"workload": "c2_tc_pl (bounded CPU sample of the same generator)", "program": PROGRAM, **s},
        "cpu_baseline": {"value": v, "unit": "tuples/s", "cores": os.cpu_count(), "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"tc_pl n={s['n']} m={s['m']} W={s['window']} alpha={s['alpha']}",
                         "full_scale": FULL_SCALE_DNF},
        "e2e": {"value": v, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
