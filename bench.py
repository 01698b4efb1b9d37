"""bench.py -- ligands docked+scored per second on B200 (BASELINE.json metric), C4 workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4] [--n N]

A step is one pass of the whole hot path over the batch:
validate -> classify -> stable bucket sort -> LPT shard -> pack -> dock every owned
bucket into every pocket -> per-pocket local top-k -> (N > 1) NCCL all_gather + merge.
`value` times it with the library HBM-resident; `e2e` times the same call from pinned
HOST buffers with the H2D copy and the D2H read of the results inside the region.
`--impl reference` times the fp64 oracle (oracle/, the paper's method written plainly)
on the host cores over a bounded sample of the same workload.
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

FLOPS_PER_EVAL = 43          # rotation 18 + fractions 3 + 7 lerps x 3 + accumulate 1
BYTES_PER_EVAL = 32          # 8 fp32 corners
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4 (SMs x FP32 lanes x FMA x max clock)
SMEM_PEAK_TBPS = 148 * 128 * 1.965e9 / 1e12          # 37.2: 128 B / clk / SM shared-memory crossbar (guide)


def measure_ceilings():
    """The roofline denominators, measured LIVE on this GPU (tools/ceilings.cu): L2 read bandwidth
    (48 MB L2-resident buffer) and random 8-corner shared-memory gathers per second."""
    import ctypes
    so = os.path.join(ROOT, "tools", "libceilings.so")
    src = os.path.join(ROOT, "tools", "ceilings.cu")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
                               "-shared", "-o", so, src])
    lib = ctypes.CDLL(so)
    lib.l2_read_gbps.restype = ctypes.c_double
    lib.l2_read_gbps.argtypes = [ctypes.c_size_t, ctypes.c_int]
    lib.smem_gather_gevals.restype = ctypes.c_double
    lib.smem_gather_gevals.argtypes = [ctypes.c_int, ctypes.c_int]
    return {"l2_read_TBps": lib.l2_read_gbps(48 << 20, 20) / 1e3,
            "gather_evals_per_s": lib.smem_gather_gevals(4096, 512) * 1e9}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--ligands", type=int, default=0, help="override the ligand count (not a bench value)")
    ap.add_argument("--poses", type=int, default=0, help="override P (sensitivity row, not a bench value)")
    ap.add_argument("--no-unsorted", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=0, help="0: geometric schedule (pipeline.chunk_bounds)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-every", type=int, default=250)
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--bucket-multiple", type=int, default=16)
    ap.add_argument("--typed", type=int, default=0,
                    help="T > 0: the per-atom-type variant (SURVEY 8(f) 4(c), Q24): typed pockets of T channels, "
                         "T atom types per ligand")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4) if len(r) > 4 + j and r[4 + j] == "Active"})
        load = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": float(np.median(load)) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def workload(args):
    import vsgen
    c = dict(vsgen.CONFIGS[args.config])
    if args.ligands:
        c["n"] = args.ligands
    if args.poses:
        c["P"] = args.poses
    lib = vsgen.ligands(c["n"], c["seed"], c["atoms"], c["rot"])
    if args.typed:
        lib.atom_type = vsgen.atom_types(lib, n_types=args.typed)
        pockets = [vsgen.typed_pocket(s, n_types=args.typed) for s in c["pockets"]]
    else:
        pockets = [vsgen.pocket(s) for s in c["pockets"]]
    rot, tr = vsgen.pose_table(c["P"])
    cs = vsgen.angle_table(c["K"])
    return c, lib, pockets, rot, tr, cs


def describe(c, args, world):
    return {"workload": f"{args.config}: {c['n']} synthetic ligands ({c['atoms'][0]}-{c['atoms'][1]} heavy atoms, "
                        f"{c['rot'][0]}-{c['rot'][1]} rotatable bonds), {len(c['pockets'])} pocket(s) 32^3 @ 1 A, "
                        f"P={c['P']} poses, K={c['K']} angle steps, S_w=1",
            "global_batch": c["n"], "n_pockets": len(c["pockets"]), "P": c["P"], "K": c["K"],
            "bucketing": "6 atom x 23 rotamer clusters (paper P:337; 4 x 21 populated)",
            "atom_types": (f"{args.typed} per-atom-type grid channels (SURVEY 8(f) 4(c), DESIGN Q24)" if args.typed
                           else "none (one grid channel)"),
            "bucket_multiple": args.bucket_multiple, "streams": args.streams,
            "parallelism": f"dp{world} (LPT bucket shards, NCCL all_gather top-k merge)" if world > 1 else "dp1",
            "l2": "inputs larger than L2 (library ~1 GB HBM-resident)"}


def run_reference(args):
    """--impl reference: the fp64 oracle on the host cores, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    c, lib, pockets, rot, tr, cs = workload(args)
    cores = os.cpu_count() or 1
    # each step docks a different bounded stratified sample (~2-4 s of CPU work on 16 cores)
    per = max(1, c["n"] // 400)
    times = []
    n_done = 0
    for s in range(args.warmup + args.steps):
        idx = np.arange(s % per, c["n"], per)[:400]
        sub = lib.subset(idx)
        t = time.perf_counter()
        for pk in pockets:
            oracle.dock_batch(sub, pk, rot, tr, cs, 1, want_xyz=False, want_debug=False, nthreads=cores)
        dt = time.perf_counter() - t
        if s >= args.warmup:
            times.append(dt)
            n_done += len(idx) * len(pockets)
    T = sum(times)
    v = n_done / T
    sample = f"{len(idx)} ligands per step (every {per}th of the {c['n']}-ligand library, offset by step), all pockets"
    print(json.dumps({
        "impl": "reference", "metric": "ligands docked+scored/sec", "value": v, "unit": "ligands/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": describe(c, args, args.gpus),
        "cpu_baseline": {"value": v, "unit": "ligands/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "ligands/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def cpu_baseline(args, c, lib, pockets, rot, tr, cs):
    import oracle
    cores = os.cpu_count() or 1
    idx = np.arange(0, c["n"], args.cpu_sample_every)
    sub = lib.subset(idx)
    t = time.perf_counter()
    for pk in pockets:
        oracle.dock_batch(sub, pk, rot, tr, cs, 1, want_xyz=False, want_debug=False, nthreads=cores)
    dt = time.perf_counter() - t
    return {"value": len(idx) * len(pockets) / dt, "unit": "ligands/s", "cores": cores, "kind": "oracle",
            "sample": f"every {args.cpu_sample_every}th ligand of the workload ({len(idx)} ligands x "
                      f"{len(pockets)} pocket(s)), fp64 full-sum oracle, {dt:.1f} s wall"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2303_06150_b200 import Engine, parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook for the multi-rank path on a one-GPU box: every rank on device 0 over gloo
    # (NCCL refuses two ranks on one GPU).  Never set for a measurement.
    single_box = os.environ.get("VSDOCK_BENCH_SAME_DEVICE") == "1"
    if single_box:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if single_box:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")

    def reduce_scalar(v, op):
        x = torch.tensor([float(v)], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(x, op=op)
        return float(x.item())

    c, lib, pockets, rot, tr, cs = workload(args)
    K_TOP = 1000
    n = lib.n

    # library HBM-resident for `value`; pinned host copies for `e2e`
    arrs = list(lib.arrays()) + ([lib.atom_type] if args.typed else [])   # (+ atom types, Q24)
    d_lib = [torch.from_numpy(a).to(dev) for a in arrs]
    h_lib = [torch.from_numpy(a).pin_memory() for a in arrs]
    h2d_bytes = sum(t.numel() * t.element_size() for t in h_lib)
    max_atoms = int(lib.n_atoms.max())

    def make_engine(na, nr):
        e = Engine(device=local, atom_clusters=na, rot_clusters=nr, bucket_multiple=args.bucket_multiple,
                   n_streams=args.streams, rank=rank, world_size=world)
        e.set_poses(rot, tr)
        e.set_angles(cs)
        ids = [e.load_pocket(p) for p in pockets]
        return e, ids

    from paper_2303_06150_b200 import VsError

    def step(e, ids, batch, on_device, host_out=None):
        failed = None
        try:
            e.submit(*batch[:7], ids, on_device=on_device, max_atoms=max_atoms,
                     atom_type=batch[7] if len(batch) > 7 else None)
            e.wait()
        except VsError as err:     # rank-local a1 error: every rank learns it from the gather
            failed = err
        tops = []
        for s in range(len(ids)):
            tops.append(parallel.global_topk(e, s, K_TOP, failed=failed))   # a10 + a11 NCCL all_gather + merge
            if host_out is not None:     # D2H of the step's per-ligand result (score, pose)
                e.results_device(s, host_out[0], host_out[1])
        return tops

    def timed(e, ids, batch, on_device, host_out=None, clocks=None):
        for _ in range(args.warmup):
            step(e, ids, batch, on_device, host_out)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dock_ms, launches, evals = [], 0, 0.0
        ctx = clocks if clocks is not None else _Null()
        with ctx:
            ev0.record(st)
            for _ in range(args.steps):
                step(e, ids, batch, on_device, host_out)
                s = e.stats()
                dock_ms.append(s["dock_ms"])
                launches += s["kernel_launches"]
                evals += s["evals_alg"]
            ev1.record(st)
            torch.cuda.synchronize()
        t = ev0.elapsed_time(ev1)
        if world > 1:
            t = reduce_scalar(t, dist.ReduceOp.MAX)
        return t, dock_ms, launches, evals

    eng, ids = make_engine(6, 23)
    clocks = Clocks(local)
    t_ms, dock_ms, launches, evals = timed(eng, ids, d_lib, True, clocks=clocks)
    ms_step = t_ms / args.steps
    value = n * len(pockets) / (ms_step / 1e3)
    # roofline of the dominant kernel (dock): algorithmic flops / dock-phase time, live CUDA events
    dock_avg = float(np.mean(dock_ms))
    evals_step = evals / args.steps
    achieved = FLOPS_PER_EVAL * evals_step / (dock_avg / 1e3) / 1e12
    # executed evaluations: the kernel also scores the identity angle (k = 0) of every moving
    # atom; algorithmic: E_alg = P (A + (K - 1) sum|M_r|)
    a_i = np.diff(lib.atom_off).astype(np.float64)
    m_i = lib.moving_per_ligand.astype(np.float64)
    K_ = c["K"]
    exec_ratio = float((a_i + K_ * m_i).sum() / max(1.0, (a_i + (K_ - 1) * m_i).sum())) if K_ > 1 else 1.0
    exec_rate = evals_step * exec_ratio / (dock_avg / 1e3)
    if world > 1:
        achieved = reduce_scalar(achieved, dist.ReduceOp.MIN)
        exec_rate = reduce_scalar(exec_rate, dist.ReduceOp.MIN)
    classes = eng.classes()
    torch.cuda.synchronize()
    ceil = measure_ceilings()          # after the timed region: live roofline denominators
    roof = min(FP32_PEAK_TFLOPS, FLOPS_PER_EVAL / BYTES_PER_EVAL * ceil["l2_read_TBps"])

    e2e = None
    if not args.no_e2e:
        # the public host-to-results API (pipeline.PipelinedDocker, PAPER.md l.200-203 double
        # buffering): pinned host CSR in, every ligand's best score / pose and the merged top-k
        # per pocket out on the host; chunk H2D copies overlap the previous chunk's docking
        from paper_2303_06150_b200.pipeline import PipelinedDocker
        eng.close()
        pdk = PipelinedDocker(device=local, n_engines=2, atom_clusters=6, rot_clusters=23,
                              bucket_multiple=args.bucket_multiple, n_streams=args.streams, rank=rank,
                              world_size=world)
        pdk.setup(rot, tr, cs, pockets)
        # geometric chunk schedule (pipeline.chunk_bounds): a small first chunk, each next one
        # up to 4x larger; a single chunk below 250k ligands (fixed per-chunk cost)
        from paper_2303_06150_b200.pipeline import chunk_bounds
        chunks = args.e2e_chunks if args.e2e_chunks > 0 else (0 if n >= 250000 else 1)
        n_chunks = len(chunk_bounds(n, chunks)) - 1
        run_e2e = lambda: pdk.run(*h_lib[:7], k=K_TOP, chunks=chunks, max_atoms=max_atoms,
                                  atom_type=h_lib[7] if len(h_lib) > 7 else None)
        for _ in range(args.warmup):
            run_e2e()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        st = torch.cuda.current_stream()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(st)
        for _ in range(args.steps):
            run_e2e()
        ev1.record(st)
        torch.cuda.synchronize()
        t_e = ev0.elapsed_time(ev1)
        if world > 1:
            t_e = reduce_scalar(t_e, dist.ReduceOp.MAX)
        pdk.close()
        nA_, nR_ = int(lib.atom_off[-1]), int(lib.frag_off[-1])
        d2h = len(pockets) * (n * 8 + nR_ + nA_ * 12 + K_TOP * 12)
        e2e = {"value": n * len(pockets) / (t_e / args.steps / 1e3), "unit": "ligands/s",
               "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h,
               "api": f"PipelinedDocker.run: pinned host CSR (general form: axes + moving-atom lists) handed to the "
                      f"C-ABI (vs_submit, on_device = 0: the library copies each chunk to the device) -> host "
                      f"best scores, poses, angle indices, best-pose coordinates (input atom order) + top-{K_TOP} "
                      f"per pocket; {n_chunks} chunk(s) {chunk_bounds(n, chunks)[1:]} over 2 engines: H2D of chunk "
                      f"i+1 and the D2H of chunk i-1's outputs under the docking of chunk i"}
    multisite = None
    if len(pockets) > 1 and not args.no_unsorted:
        # the same step with the fused multi-site cluster launches (records
        # staged once per cluster) instead of one launch per pocket
        if args.no_e2e:
            eng.close()
        pe = Engine(device=local, atom_clusters=6, rot_clusters=23, bucket_multiple=args.bucket_multiple,
                    n_streams=args.streams, rank=rank, world_size=world, fused_sites=True)
        pe.set_poses(rot, tr)
        pe.set_angles(cs)
        pids = [pe.load_pocket(p) for p in pockets]
        t_p, dock_p, _, _ = timed(pe, pids, d_lib, True)
        pv = n * len(pockets) / (t_p / args.steps / 1e3)
        multisite = {"fused_value": pv, "per_pocket_value": value, "unit": "ligand-pockets/s",
                     "fused_over_per_pocket": pv / value, "fused_dock_ms_per_step": float(np.mean(dock_p)),
                     "per_pocket_dock_ms_per_step": dock_avg,
                     "note": "fused = thread-block clusters of one CTA per pocket, each ligand round staged once per "
                             "cluster by multicast TMA (cluster size chosen by cudaOccupancyMaxActiveClusters); the "
                             "default (value) is one persistent launch per (class, pocket)"}
        pe.close()
    unsorted = None
    if not args.no_unsorted:
        if args.no_e2e and multisite is None:
            eng.close()
        ue, uids = make_engine(1, 1)
        t_u, dock_u, _, _ = timed(ue, uids, d_lib, True)
        uv = n * len(pockets) / (t_u / args.steps / 1e3)
        unsorted = {"value": uv, "unit": "ligands/s", "dock_ms_per_step": float(np.mean(dock_u)),
                    "bucketed_over_unsorted": value / uv}
        ue.close()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, c, lib, pockets, rot, tr, cs)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "dock_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            if tj.get("config") == args.config and tj.get("n") == n:
                traffic = tj.get("dram_bytes_per_dock_phase")
        except Exception:
            traffic = None
    if rank == 0:
        line = {
            "metric": "ligands docked+scored/sec", "value": value, "unit": "ligands/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": describe(c, args, world),
            "roofline": {"bound": "alu", "achieved": achieved, "peak": roof, "unit": "TFLOP/s",
                         "frac": achieved / roof, "traffic": traffic,
                         "kernel": "dock_kernel<AC,NW,PPW,GM,K> (all launches of the dock phase)",
                         "peak_source": "BASELINE.json's 'FP32/L2 roofline' (SURVEY 8(d)): min(FP32 peak, 43/32 "
                                        "flop/B x L2 read bandwidth measured live in this run by tools/ceilings.cu); "
                                        "FP32 peak = 148 SMs x 128 lanes x 2 x 1.965 GHz (guide unit counts)",
                         "dock_ms_per_step": dock_avg, "evals_per_step": evals_step,
                         "flops_per_eval": FLOPS_PER_EVAL, "l2_read_TBps_measured": ceil["l2_read_TBps"],
                         "fp32": {"peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS},
                         "smem": {"bound": "smem", "unit": "TB/s",
                                  "achieved": achieved / FLOPS_PER_EVAL * BYTES_PER_EVAL,
                                  "peak": SMEM_PEAK_TBPS,
                                  "frac": achieved / FLOPS_PER_EVAL * BYTES_PER_EVAL / SMEM_PEAK_TBPS,
                                  "bytes_per_eval": BYTES_PER_EVAL,
                                  "executed_evals_per_s": exec_rate,
                                  "random_gather_ceiling_evals_per_s": ceil["gather_evals_per_s"],
                                  "frac_of_gather_ceiling": exec_rate / ceil["gather_evals_per_s"],
                                  "note": "8 fp32 corner gathers per evaluation from the shared-memory grid; random "
                                          "4-byte gathers run ~3-way bank-conflicted, so the gather ceiling (measured "
                                          "live, uniformly random points) is ~1/3.5 of the crossbar peak"}},
            "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": launches,
            "cpu_baseline": cpu, "unsorted": unsorted, "multisite": multisite,
            "classes": [{k: cl[k] for k in ("kernel_atoms", "warps_per_cta", "regs_per_thread", "dyn_smem", "blocks_per_sm",
                                            "ligands_per_cta", "l", "capacity")} for cl in classes],
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


if __name__ == "__main__":
    main()
