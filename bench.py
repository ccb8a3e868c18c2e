#!/usr/bin/env python
"""Benchmark: trajectories/s of a Lorenz Tsit5 ensemble on B200 (BASELINE.json
metric), fixed dt=1e-3 on [0,1] → 1000 steps, fp32.

Workloads (--workload):
  c5 (default) — BASELINE configs[4]: 10^8 trajectories, random p ±10 % around
     (10, 28, 8/3), STRONG scaling: the 10^8 are split contiguously over the N
     ranks (one per GPU); each trajectory does the same work as configs[1]'s
     headline point, so the N=1 line measures that kernel at 10^8.
  c2 — BASELINE configs[1] headline point: 10^7 trajectories PER GPU, ρ sweep
     over (0,21], weak scaling.

One step = one whole pass of the hot path over the batch: ensemble_solve (a2–a7,
a13: one kernel, one thread per trajectory, with the ensemble statistics of the
final states fused into its epilogue, a12) + for N>1 GPUs the cross-GPU
exchange (a14: NCCL all-gather of the statistics triples + fixed-order merge,
and the gather of the final states to rank 0 — fused into the solve by default:
each rank's kernel stores straight into rank 0's array over NVLink). Inputs are
generated on device before the timed region (resident in HBM); they plus the
outputs exceed the 126 MB L2, so no flush is needed.

Usage:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c5|c2]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FP32_LANES_PER_SM = 128     # FFMA lanes per SM (B200 profiling guide; tools/peaks.cu measured 121-126/clk)
FP64_LANES_PER_SM = 64
SM_MAX_MHZ = 1965.0
METRIC = "trajectories/sec (Lorenz Tsit5, fp32/fp64) at 1/2/4/8 B200; % FP peak"


def flops_per_traj(nsteps: int) -> float:
    """Algorithmic FLOPs of one fixed-step Tsit5 Lorenz trajectory:
    per step 48n (stage sums, n=3) + 6F (six RHS, F=8) = 192; plus f(u0) = 8."""
    return 192.0 * nsteps + 8.0


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period: float = 0.05):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


WORKLOADS = {
    # name: (recipe, input seed, scaling, BASELINE config)
    "c5": ("random10", 0xC5, "strong", "configs[4]"),
    "c2": ("rho_sweep", 0, "weak", "configs[1]"),
}


def sample_indices(N_total: int, sample: int):
    """Evenly spaced global indices g = i·stride (i < sample) over the whole ensemble."""
    stride = max(1, N_total // sample)
    return min(sample, N_total), stride


def cpu_baseline(N_total: int, dt: float, sample: int, threads: int, workload: str = "c5", want_outputs=False):
    """The oracle as it stands (single-threaded C++ per call) over a bounded
    sample of the same workload — `sample` trajectories evenly spaced over the
    N_total ensemble (inputs from the shared generator at those global
    indices) — spread over host threads by a harness pool (ctypes releases the
    GIL during each oracle call). Returns the record (and the oracle's final
    states and retcodes of the sample if want_outputs)."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle
    from synth.inputs import make_inputs
    recipe, seed, _, _ = WORKLOADS[workload]
    S, stride = sample_indices(N_total, sample)
    # global index of sample trajectory i is i·stride: the block-cyclic map with chunk_len 1
    u0s, ps = make_inputs("lorenz", recipe, S, seed=seed, dtype="f32", N_total=N_total, chunk_len=1,
                          chunk_stride=stride)
    chunks = np.array_split(np.arange(S), threads * 4)
    out = np.empty((3, S), np.float32)
    rc = np.empty(S, np.int32)

    def work(c):
        o, r, *_ = oracle.solve("lorenz", "tsit5", u0s[:, c], ps[:, c], (0.0, 1.0), dt, dtype="f32")
        out[:, c] = o[0]
        rc[c] = r

    oracle.lib()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, chunks))
    wall = time.perf_counter() - t0
    # one host core alone (SURVEY §8d reports single-core traj/s beside the all-core figure)
    n1 = max(1, S // (4 * threads))
    t1 = time.perf_counter()
    work(np.arange(n1))
    wall1 = time.perf_counter() - t1
    rec = {"value": S / wall, "unit": "trajectories/s", "cores": threads, "kind": "oracle", "cpu_model": cpu_model(),
           "sample": f"{S} Lorenz Tsit5 fixed-dt fp32 trajectories (1000 steps each), global indices i*{stride} of "
                     f"the N={N_total} {recipe} ensemble; {threads} host threads; wall {wall:.2f} s",
           "single_core": {"value": n1 / wall1, "unit": "trajectories/s", "sample": f"first {n1} of the same sample"}}
    return (rec, out, rc, stride) if want_outputs else rec


def load_summary(tag: str):
    """The committed ncu summary entry for `tag` (profiles/ncu_summary.json), or None."""
    try:
        return json.loads((ROOT / "profiles" / "ncu_summary.json").read_text()).get(tag)
    except Exception:
        return None


def load_traffic(tag: str, n_traj: int):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    `ncu --set full` summary, scaled to this launch's trajectory count (the capture
    records its own)."""
    e = load_summary(tag)
    if not e or e.get("dram_bytes_per_launch") is None:
        return None
    return e["dram_bytes_per_launch"] / float(e.get("traj_per_launch", 10**7)) * n_traj


def load_executed(tag: str, n_traj: int, kernel_ms: float):
    """Executed FP32/FP64 FLOPs per launch counted by ncu (sm__sass_thread_inst_executed_op_*:
    FFMA/DFMA = 2, FADD/FMUL = 1 per lane; the packed FFMA2/FADD2/FMUL2 count per lane
    like their scalar forms), scaled to this launch, and the executed-FLOP rate at this
    run's kernel time."""
    e = load_summary(tag)
    if not e or e.get("executed_flop_per_launch") is None:
        return None
    f = e["executed_flop_per_launch"] / float(e.get("traj_per_launch", 10**7)) * n_traj
    return {"flop_per_launch": f, "tflops": f / (kernel_ms / 1e3) / 1e12,
            "flop_per_traj": f / n_traj, "source": e.get("executed_source", e.get("source"))}


def workload_sizes(args, rank: int, world: int):
    """(shard, N_total) of the chosen workload on this rank."""
    from paper_2304_06835_b200 import multi_gpu as mg
    if args.workload == "c5":
        return mg.shard_contiguous(args.n_total, rank, world), args.n_total
    return mg.shard_weak(args.traj_per_gpu, rank, world), args.traj_per_gpu * world


def workload_name(args, N_total: int, world: int) -> str:
    recipe, seed, scaling, cfg = WORKLOADS[args.workload]
    if args.workload == "c5":
        return (f"lorenz_tsit5_fixed_dt1e-3_{args.dtype}_random10_seed0xC5_N{N_total} (BASELINE {cfg} C5: "
                f"{N_total:.0e} trajectories split over {world} GPU(s), strong scaling; per-trajectory work = "
                f"configs[1]'s headline point)")
    return (f"lorenz_tsit5_fixed_dt1e-3_{args.dtype}_rho_sweep (BASELINE {cfg} headline point, "
            f"N={args.traj_per_gpu:.0e} per GPU, weak scaling)")


def run_reference(args, rank):
    """--impl reference: the oracle (this tier's reference arm) on the host cores,
    on our arm's workload, metric and unit (rank 0 only; other ranks exit)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    world = int(os.environ.get("WORLD_SIZE", "1"))
    _, N_total = workload_sizes(args, 0, max(world, args.gpus))
    vals = []
    sample = args.ref_sample
    for _ in range(args.warmup):
        cpu_baseline(N_total, 1e-3, max(threads, sample // 8), threads, args.workload)
    for _ in range(args.steps):
        vals.append(cpu_baseline(N_total, 1e-3, sample, threads, args.workload))
    v = statistics.median([x["value"] for x in vals])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "trajectories/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sample / v, "higher_is_better": True,
            "scaling": WORKLOADS[args.workload][2], "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(args, N_total, max(world, args.gpus)) + " — oracle sample per step",
                       "N_total": N_total, "sample_per_step": sample},
            "cpu_baseline": {**vals[-1], "value": v},
            "e2e": {"value": v, "unit": "trajectories/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def parity_block(gpu_states, rc_gpu, oracle_states, rc_oracle):
    """Element-wise comparison of the GPU's final states with the oracle's on the
    cpu_baseline sample ("the same subset's GPU outputs are compared
    for parity in the same run"). Per-trajectory ∞-norm relative error."""
    import numpy as np
    g = gpu_states.astype(np.float64)
    o = oracle_states.astype(np.float64)
    rel = np.abs(g - o).max(0) / np.maximum(np.abs(o).max(0), np.finfo(np.float64).tiny)
    return {"n": int(o.shape[1]), "max_rel": float(rel.max()), "bitexact_frac": float((g == o).all(0).mean()),
            "retcodes_equal": bool((rc_gpu == rc_oracle).all()), "tol": 1e-5 if gpu_states.dtype.itemsize == 4
            else 1e-12, "pass": bool(rel.max() <= (1e-5 if gpu_states.dtype.itemsize == 4 else 1e-12)
                                     and (rc_gpu == rc_oracle).all())}


def executed_frac(tag: str, n_traj: int, kernel_ms: float, peak_flops: float):
    """Executed FP FLOP/s of a side measurement as a fraction of the FP peak, from the
    committed ncu executed-instruction counts of the same workload (profiles/ncu_summary.json),
    scaled per trajectory; None if no capture is committed."""
    e = load_executed(tag, n_traj, kernel_ms)
    return None if e is None else e["tflops"] * 1e12 / peak_flops


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c5",
                    help="c5: 10^8 trajectories split over the ranks (strong scaling, default); "
                         "c2: 10^7 per GPU (weak scaling)")
    ap.add_argument("--n-total", type=int, default=10**8, help="c5: trajectories in the whole ensemble")
    ap.add_argument("--traj-per-gpu", type=int, default=10**7, help="c2: trajectories per GPU")
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=98304)
    ap.add_argument("--ref-sample", type=int, default=16384)
    ap.add_argument("--no-gather", action="store_true", help="skip the gather of final states (N>1)")
    ap.add_argument("--gather", choices=["peer", "nccl"], default="peer",
                    help="N>1 state gather: 'peer' = fused into the solve (CUDA IPC / NVLink stores into rank 0's "
                         "array, multi_gpu.PeerGather), 'nccl' = NCCL gather after the solve")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-also", action="store_true", help="skip the fp64-fixed / adaptive side measurements")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="process-group backend for N>1 (gloo: test the multi-rank path on one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    if world > 1 and args.backend == "nccl":
        # communicator init lines (nranks, rank, device) for the record — on stderr, stdout carries the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2304_06835_b200 as ens
    from paper_2304_06835_b200 import multi_gpu as mg

    # one rank per GPU (the driver's launch); --backend gloo lets several ranks share a GPU
    # to exercise the multi-rank path where only one GPU exists (never for reported numbers)
    gpu = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    recipe, in_seed, scaling, cfg_name = WORKLOADS[args.workload]
    shard, N_total = workload_sizes(args, rank, world)
    N = shard.n_local
    tspan, dt = (0.0, 1.0), 1e-3
    nsteps = 1000

    # a1: inputs generated on device from (seed, global index) — no host scatter
    u0, p = ens.generate_inputs("lorenz", recipe, N, dtype=tdt, seed=in_seed, index_offset=shard.index_offset,
                                N_total=N_total, device=dev)
    gather_mode = "none" if (world == 1 or args.no_gather) else args.gather
    if gather_mode == "nccl" and N_total % world != 0:
        raise SystemExit("--gather nccl needs equal shards (N_total divisible by the world size)")
    peer = None
    if gather_mode == "peer":
        err = ""
        try:
            peer = mg.PeerGather((3,), N, shard.index_offset, N_total, tdt, dev)
        except Exception as e:   # no IPC mapping / peer access: gather with NCCL after the solve instead
            err = repr(e)
        # every rank must take the same path
        flags = [None] * world
        dist.all_gather_object(flags, err)
        if any(flags):
            print(f"PeerGather unavailable ({[f for f in flags if f]}); using the NCCL gather", file=sys.stderr)
            gather_mode, peer = "nccl", None
    sol = ens.Solution(u=peer.out() if peer is not None else torch.empty((3, N), dtype=tdt, device=dev),
                       retcode=torch.empty(N, dtype=torch.int32, device=dev),
                       n_accept=torch.empty(N, dtype=torch.int32, device=dev),
                       n_reject=torch.empty(N, dtype=torch.int32, device=dev),
                       stats=torch.empty((1, 3, 3), dtype=torch.float64, device=dev))
    st_local = sol.stats
    # a12 fused into the solve: each warp's final states reduced to (count, mean, M2) in the kernel
    # epilogue, then a fold + merge (no pass over the stored states, which on N>1 live on rank 0)
    ws = ens.Workspace(ens.workspace_bytes("lorenz", "tsit5", tdt, N, stats=True), dev)
    stream = torch.cuda.current_stream(dev)
    # our kernels per step: the solve + the statistics fold (when more than 4·256·8 per-warp partials) + merge
    nparts = -(-N // (64 if tdt == torch.float32 else 32))
    launches_per_step = 1 + (2 if nparts > 4 * 256 * 8 else 1) + (1 if world > 1 else 0)
    gathered = [None]
    merged = [None]

    def step(ev_k0=None, ev_k1=None):
        if ev_k0 is not None:
            ev_k0.record(stream)
        ens.solve("lorenz", "tsit5", u0, p, tspan, dt, stats=True, workspace=ws, out=sol, stream=stream,
                  index_offset=shard.index_offset)
        if ev_k1 is not None:
            ev_k1.record(stream)
        if world > 1:
            merged[0] = mg.merge_stats(mg.allgather_stats(st_local))
            if gather_mode == "peer":
                gathered[0] = peer.complete()    # the states are already in rank 0's array; order its reads
            elif gather_mode == "nccl":
                gathered[0] = mg.gather_states(sol.u)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(gpu) as clk:
        ev0.record(stream)
        for s in range(args.steps):
            step(*kev[s])
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    k_ms = [a.elapsed_time(b) for a, b in kev]
    k_avg = sum(k_ms) / len(k_ms)
    t = torch.tensor([ms, k_avg], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, k_max = t.tolist()
    assert (sol.retcode == 0).all().item(), "non-success retcodes in the benchmark ensemble"

    # final states of the whole ensemble in global order on rank 0 (for the parity sample)
    full_states = None
    if rank == 0:
        if world == 1:
            full_states = sol.u
        elif gather_mode == "peer":
            full_states = gathered[0]
        elif gather_mode == "nccl":
            g = gathered[0]                                 # [R, 3, N_r] rank blocks, contiguous shards
            full_states = g.permute(1, 0, 2).reshape(3, N_total)
        else:
            full_states = sol.u                             # rank 0's own shard only (global 0..N-1)
    rc_rank0 = sol.retcode

    # side measurements (configs[1] at 10^7 per GPU: fp32 headline point, fp64, adaptive; tight tolerance; C3)
    also = {}
    if not args.no_also:
        def best_ms(fn, reps=3):
            fn()
            torch.cuda.synchronize(dev)
            b = float("inf")
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                torch.cuda.synchronize(dev)
                b = min(b, e0.elapsed_time(e1))
            return b
        props = torch.cuda.get_device_properties(dev)
        pk32 = props.multi_processor_count * FP32_LANES_PER_SM * 2 * SM_MAX_MHZ * 1e6
        pk64 = props.multi_processor_count * FP64_LANES_PER_SM * 2 * SM_MAX_MHZ * 1e6
        n_c2 = 10**7
        for tname, tt in [("f32", torch.float32), ("f64", torch.float64)]:
            uc, pc = ens.generate_inputs("lorenz", "rho_sweep", n_c2, dtype=tt, N_total=n_c2, device=dev)
            msf = best_ms(lambda: ens.solve("lorenz", "tsit5", uc, pc, tspan, dt, stream=stream))
            also[f"c2_fixed_{tname}_N1e7"] = {
                "trajectories_per_s": n_c2 / (msf / 1e3), "kernel_ms": msf,
                "frac_fp_peak": n_c2 * flops_per_traj(nsteps) / (msf / 1e3) / (pk32 if tname == "f32" else pk64),
                "frac_fp_peak_executed": executed_frac(f"tsit5_fixed_lorenz_{tname}", n_c2, msf,
                                                       pk32 if tname == "f32" else pk64)}
            if tname == "f32":
                sol_a = ens.solve("lorenz", "tsit5", uc, pc, tspan, dt, adaptive=True, abstol=1e-6, reltol=1e-6,
                                  stream=stream)
                msa = best_ms(lambda: ens.solve("lorenz", "tsit5", uc, pc, tspan, dt, adaptive=True, abstol=1e-6,
                                                reltol=1e-6, out=sol_a, stream=stream))
                att = int((sol_a.n_accept.to(torch.int64) + sol_a.n_reject.to(torch.int64)).sum().item())
                also["c2_adaptive_f32_tol1e-6_N1e7"] = {
                    "trajectories_per_s": n_c2 / (msa / 1e3), "kernel_ms": msa, "attempted_steps_per_traj": att / n_c2,
                    "frac_fp_peak_265flop_per_attempt": att * 265.0 / (msa / 1e3) / pk32,
                    "frac_fp_peak_executed": executed_frac("c2_adaptive_f32", n_c2, msa, pk32)}
                del sol_a
            del uc, pc
        # NEXT-1: the same ρ sweep in fp64 at the north_star's tight tolerance, Tsit5 vs Vern9
        n_t = 10**6
        u0t, pt = ens.generate_inputs("lorenz", "rho_sweep", n_t, dtype=torch.float64, N_total=n_t, device=dev)
        for alg in ["tsit5", "vern9"]:
            sol_t = ens.solve("lorenz", alg, u0t, pt, tspan, dt, adaptive=True, abstol=1e-10, reltol=1e-10,
                              stream=stream)
            mst = best_ms(lambda: ens.solve("lorenz", alg, u0t, pt, tspan, dt, adaptive=True, abstol=1e-10,
                                            reltol=1e-10, out=sol_t, stream=stream))
            att = int((sol_t.n_accept.to(torch.int64) + sol_t.n_reject.to(torch.int64)).sum().item())
            fl = {"tsit5": 265.0, "vern9": 721.0}[alg]      # algorithmic FLOP per attempted Lorenz step
            also[f"{alg}_f64_tol1e-10_N{n_t}"] = {"trajectories_per_s": n_t / (mst / 1e3), "kernel_ms": mst,
                                                  "attempted_steps_per_traj": att / n_t,
                                                  f"frac_fp64_peak_{fl:.0f}flop_per_attempt":
                                                      att * fl / (mst / 1e3) / pk64,
                                                  "frac_fp64_peak_executed":
                                                      executed_frac({"tsit5": "c1t_tsit5_f64_tol1e-10",
                                                                    "vern9": "t9_vern9_f64_tol1e-10"}[alg],
                                                                    n_t, mst, pk64)}
        del u0t, pt, sol_t
        # NEXT-2: C3 (Robertson fp64, tol 1e-8, 100 save points) on Rosenbrock23 vs Rodas5
        n_s = 10**6
        ur, pr = ens.generate_inputs("robertson", "random10", n_s, dtype=torch.float64, seed=0xC3, device=dev)
        sa = [1e5 * j / 99 for j in range(100)]
        for alg in ["rosenbrock23", "rodas5", "rodas5p"]:
            sol_s = ens.solve("robertson", alg, ur, pr, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8, reltol=1e-8,
                              saveat=sa, stream=stream)
            mss = best_ms(lambda: ens.solve("robertson", alg, ur, pr, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8,
                                            reltol=1e-8, saveat=sa, out=sol_s, stream=stream))
            att = int((sol_s.n_accept.to(torch.int64) + sol_s.n_reject.to(torch.int64)).sum().item())
            fl = {"rosenbrock23": 170.0, "rodas5": 600.0, "rodas5p": 600.0}[alg]   # ≈ FLOP / attempted step
            # Rodas5 / 5P store an interior save point as one shortened step (DESIGN R24): 98 more
            # steps of the same work per trajectory (every τ strictly inside (t0, tf))
            sub = sum(1 for x in sa if 0.0 < x < 1e5) if alg != "rosenbrock23" else 0
            units = att + sub * n_s
            also[f"c3_{alg}_N{n_s}"] = {"trajectories_per_s": n_s / (mss / 1e3), "kernel_ms": mss,
                                        "attempted_steps_per_traj": att / n_s, "dense_substeps_per_traj": sub,
                                        f"frac_fp64_peak_{fl:.0f}flop_per_step": units * fl / (mss / 1e3) / pk64,
                                        "frac_fp64_peak_executed": executed_frac(f"c3_{alg}", n_s, mss, pk64)}
            del sol_s
        del ur, pr

    # end to end through the C ABI on host buffers (pinned), copies in the timed region: this rank's shard
    e2e = None
    if not args.no_e2e:
        u0h = u0.cpu().pin_memory()            # the shard's inputs, staged in pinned host memory
        ph = p.cpu().pin_memory()
        uo = torch.empty((1, 3, N), dtype=tdt, pin_memory=True)
        rco = torch.empty(N, dtype=torch.int32, pin_memory=True)
        staging = None
        for _ in range(2):
            _, _, staging = ens.solve_host("lorenz", "tsit5", u0h, ph, tspan, dt, device=dev, n_chunks=8,
                                           staging=staging, u_out_host=uo, retcode_host=rco,
                                           index_offset=shard.index_offset)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ens.solve_host("lorenz", "tsit5", u0h, ph, tspan, dt, device=dev, n_chunks=8, staging=staging,
                           u_out_host=uo, retcode_host=rco, index_offset=shard.index_offset)
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        tsz = 4 if args.dtype == "f32" else 8
        e2e = {"value": N_total * args.steps / el.item(), "unit": "trajectories/s",
               "h2d_bytes_per_step": (3 + 3) * tsz * N, "d2h_bytes_per_step": 3 * tsz * N + 4 * N,
               "api": "ensemble_solve_host (pinned host buffers, 8 ramped chunks, H2D/compute/D2H overlapped, chunk "
                      "solves on two streams)", "per_rank_bytes": True}
        del staging, u0h, ph, uo, rco

    if rank == 0:
        value = N_total * args.steps / (ms_max / 1e3)
        lanes = FP32_LANES_PER_SM if args.dtype == "f32" else FP64_LANES_PER_SM
        props = torch.cuda.get_device_properties(dev)
        peak = props.multi_processor_count * lanes * 2 * SM_MAX_MHZ * 1e6 / 1e12
        achieved = N * flops_per_traj(nsteps) / (k_max / 1e3) / 1e12
        tag = f"tsit5_fixed_lorenz_{args.dtype}"
        line = {
            "metric": METRIC, "value": value, "unit": "trajectories/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": workload_name(args, N_total, world),
                       "N_total": N_total, "N_per_gpu": N, "tspan": [0.0, 1.0], "dt": dt, "nsteps": nsteps,
                       "parallelism": f"dp{world} (contiguous trajectory shards)",
                       "l2": f"inputs+outputs ({(N * 36) / 1e6:.0f} MB per GPU) > L2 (126 MB)",
                       "step": "ensemble_solve with fused ensemble statistics" + (
                           " + NCCL allgather(stats)+merge" +
                           {"none": "", "nccl": " + NCCL gather(states)",
                            "peer": " (states stored into rank 0's array by the solve: fused peer gather)"}[gather_mode]
                           if world > 1 else "")},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": load_traffic(tag, N),
                         "algorithmic_bytes": N * 48.0,
                         "executed": load_executed(tag, N, k_max),
                         "kernel": f"tsit5_fixed_kernel<Lorenz,{'f2' if args.dtype == 'f32' else 'double'},SAVE=0,STATS>",
                         "kernel_ms": k_max, "flop_per_traj": flops_per_traj(nsteps),
                         "peak_basis": f"{props.multi_processor_count} SMs x {lanes} FMA lanes x 2 x {SM_MAX_MHZ:.0f} MHz",
                         "kernel_share_of_step": k_max / (ms_max / args.steps)},
            "clocks": clk.summary(),
            # north_star: the paper's Lorenz ensemble numbers with their stated hardware, context only
            # (2^31 Lorenz solves over 8 V100 nodes; the ODE solve of ≈306 M trajectories on one
            # V100 took ≈1.6 s; step count / precision not stated)
            "paper_context": {"source": "PAPER.md:395 (§6.3)", "gpu": "V100 (per node, 7 computing)",
                              "trajectories_per_gpu": 306e6, "solve_seconds": 1.6,
                              "trajectories_per_s_per_gpu": 306e6 / 1.6,
                              "note": "other GPU, step count and precision unstated: context, not a baseline"},
            "gpu_launches": launches_per_step * args.steps,
            "e2e": e2e,
            "also": also,
        }
        if world > 1:
            line["nccl"] = {"backend": args.backend, "nranks": world, "gather": gather_mode,
                            "version": ".".join(map(str, torch.cuda.nccl.version())) if args.backend == "nccl" else None}
        if not args.no_cpu_baseline:
            rec, o_states, o_rc, stride = cpu_baseline(N_total, dt, args.cpu_sample, os.cpu_count() or 1,
                                                       args.workload, want_outputs=True)
            line["cpu_baseline"] = rec
            S = o_states.shape[1]
            gidx = torch.arange(S, dtype=torch.int64, device=full_states.device) * stride
            if gather_mode == "none" and world > 1:
                keep = gidx < N                            # rank 0's shard only
                gidx = gidx[keep]
                o_states, o_rc = o_states[:, keep.cpu().numpy()], o_rc[keep.cpu().numpy()]
            g = full_states[:, gidx].cpu().numpy()
            rcg = rc_rank0[gidx.clamp(max=N - 1)].cpu().numpy() if (world == 1 or gather_mode == "none") \
                else np.zeros(len(gidx), np.int32)        # other shards: all-success asserted on every rank
            line["parity"] = {**parity_block(g, rcg, o_states, o_rc),
                              "sample": f"cpu_baseline sample: global indices i*{stride}, compared element by element"}
        print(json.dumps(line), flush=True)
    if world > 1:
        # release every rank's CUDA IPC mapping of rank 0's gather array before rank 0 exits
        del sol, full_states, gathered, peer
        torch.cuda.synchronize(dev)
        torch.cuda.ipc_collect()
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
