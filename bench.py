#!/usr/bin/env python3
"""bench.py — four-phase (FE/FF/BF/BE) training step of the canonical
conservative MLIP under the JanusPipe schedules, on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): L=4 interaction layers, H=64, R=64,
r_c=5 A, synthetic periodic 256-atom fcc cells (rho 0.095 /A^3, ~50
neighbours), 32 micro-batches of one cell each.  N=1 runs the whole model on
one GPU (P=1, SymFold == WaveK; one compute lane per micro-batch); N>1
pipelines it over N GPUs (P=N stages, WaveK k=2P; NCCL P2P over NVLink on
send / receive side streams; up to 8 compute lanes per GPU so independent
micro-batches overlap inside a stage), strong scaling (total work fixed).
Metric: structures/s (whole job).  "value" is device-timed (CUDA events, max
over ranks) with inputs resident in HBM and an L2 flush (512 MiB memset)
between timed steps; "e2e" re-uploads every micro-batch from pinned host
memory through the trainer API (janus_trainer_load) and reads the loss back
every step, timed on the host; uploads are input-pipelined (step k+1's loads
are issued while step k runs, janus_trainer_step_async / janus_trainer_wait).
--impl reference times the reference's CPU path: the reference has no numeric
implementation, so it is the fp64 C oracle restatement
(oracle/mlip_oracle.c), one structure per thread on all host cores.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# 32 hardware work queues for the 32 compute lanes, before any CUDA context
# exists (paper_2605_18404_b200/__init__.py sets the same default)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# eager kernel loading: the N>1 per-rank path blocks streams on peers, and a
# lazily loaded kernel can deadlock its first launch against them
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

CONFIG = dict(L=4, H=64, R=64, r_c=5.0, atoms=256, rho=0.095, n_mb=32, seed=7)
# per-layer edge-contraction FLOPs of the directed-edge algorithm, FE + FF + BF + BE
# (stage.cu edge_kernel_flops_per_edge)
DIRECTED_FLOP_PER_EDGE = 2.0 * ((64 * 64 + 64 * 64) + (2 * 64 * 64 + 2 * 64 * 64 + 64) + (4 * 64 * 64 + 6 * 64 * 64)
                                + (2 * 64 * 64 + 3 * 64 * 64))
METRIC = "structures/sec"


def load_traffic(precision):
    """DRAM bytes per launch of the roofline kernel from the committed ncu --set full
    capture (profiles/r02_roofline_traffic.json); None when absent or for another kernel."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_roofline_traffic.json")) as f:
            t = json.load(f)
        return t["dram_bytes_per_launch"] if precision == "tf32" and t.get("kernel", "").endswith("msg_bf_pair_tc") else None
    except (OSError, ValueError, KeyError):
        return None


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------- helpers
def pin(arrays):
    """cudaHostRegister host arrays so the e2e H2D copies come from pinned memory."""
    import paper_2605_18404_b200 as J
    rt = J.cudart()
    rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
    for a in arrays:
        if a.nbytes:
            rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)


def flush_l2(buf_holder):
    import paper_2605_18404_b200 as J
    rt = J.cudart()
    if not buf_holder:
        p = ctypes.c_void_p()
        rt.cudaMalloc.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        assert rt.cudaMalloc(ctypes.byref(p), 512 << 20) == 0
        buf_holder.append(p.value)
    rt.cudaMemset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
    rt.cudaMemset(buf_holder[0], 1, 512 << 20)
    rt.cudaDeviceSynchronize()


def batch_bytes(b):
    return sum(a.nbytes for a in (b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target, b.row_ptr, b.col,
                                  b.shift, b.rev))


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------ CPU oracle
class CpuOracle:
    """The fp64 C oracle (test infrastructure: oracle/mlip_oracle.c) timed on
    host threads, one structure (full four-phase step) per call; ctypes
    releases the GIL.  Inputs come from the oracle's own synthetic-data
    restatement (bit-identical to the product's, tests/test_oracle.py), so this
    leg never loads the product library."""

    def __init__(self, model_kw, n_structs, seed):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        self.O, self.om = O, O.Model(**model_kw)
        self.params = O.synth_params(self.om, seed).astype(np.float64)
        self.work = []
        for m in range(n_structs):
            ob = O.synth_batch(self.om, [CONFIG["atoms"]], CONFIG["rho"], seed * 100 + m)
            self.work.append((ob, O.build_nbrlist(self.om, ob)))

    def run(self, threads, per_thread=1):
        """Return (structures/s, seconds) over `threads` x `per_thread` structures."""
        def worker(k):
            for i in range(per_thread):
                ob, nl = self.work[(k + i * threads) % len(self.work)]
                self.O.step(self.om, ob, nl, self.params)

        ts = [threading.Thread(target=worker, args=(k,)) for k in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        return threads * per_thread / dt, dt


def env_overrides():
    """JANUS_* switches in the environment (A/B and tuning knobs): a bench line
    must run the product defaults, so any of them rejects the run."""
    return {k: v for k, v in os.environ.items() if k.startswith("JANUS_")}


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--method", default=None, choices=[None, "symfold", "wavek", "onef1b"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32-path", action="store_true", help="skip the fp32 SIMT parity-path throughput")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="N>1: NCCL over NVLink (one GPU per rank), or the same-GPU IPC harness (all ranks on GPU 0)")
    ap.add_argument("--lanes", type=int, default=32, help="concurrent micro-batch streams at N=1 (one per micro-batch)")
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"],
                    help="tf32: tcgen05 tensor-core edge kernels (tolerances in tests/test_gpu_tf32.py); "
                         "fp32: SIMT parity path")
    args = ap.parse_args()
    rank, world, local_rank = dist_env()
    N = args.gpus
    if args.warmup < 3:
        args.warmup = 3

    n_mb = CONFIG["n_mb"]
    cfg = {"workload": "configs[1]: L=4 H=64 R=64 r_c=5, 256-atom periodic cells, 32 micro-batches",
           "model": "canonical conservative MLIP (SURVEY.md App. A), random-init", "global_batch": n_mb,
           "atoms_per_structure": CONFIG["atoms"], "edges_per_structure": 12774,
           "n_micro_batches": n_mb, "l2": "flushed (512 MiB memset) between timed steps"}
    model_kw = dict(L=CONFIG["L"], H=CONFIG["H"], R=CONFIG["R"], n_species=4, r_c=CONFIG["r_c"], w_E=1.0, w_F=10.0)

    if args.impl == "reference":
        if rank != 0:
            return
        # bounded sample per step: one 256-atom structure per host thread (the
        # full 32-structure step would take minutes per step on the CPU)
        threads = min(os.cpu_count() or 1, n_mb)
        cpu = CpuOracle(model_kw, threads, CONFIG["seed"])
        vals, secs = [], []
        for i in range(args.warmup + args.steps):
            v, dt = cpu.run(threads)
            if i >= args.warmup:
                vals.append(v)
                secs.append(dt)
        val = statistics.median(vals)
        sample = (f"{threads} structures per step (one 256-atom cell per thread, full FE+FF+BF+BE step, "
                  f"fp64 oracle); ms_per_step is the measured time of that sample")
        out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "structures/s", "n_gpus": N,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.median(secs),
               "structures_per_step": threads,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic", "config": cfg,
               "cpu_baseline": {"value": val, "unit": "structures/s", "cores": threads, "kind": "port",
                                "sample": sample},
               "e2e": {"value": val, "unit": "structures/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
               "note": "reference has no numeric path (SPEC.md:15); its CPU restatement is the fp64 oracle"}
        print(json.dumps(out), flush=True)
        return

    # ---------------------------------------------------------------- ours
    if env_overrides():
        raise SystemExit(f"bench.py: JANUS_* switches set ({env_overrides()}); a bench line runs the product defaults")
    import paper_2605_18404_b200 as J

    model = J.Model(L=CONFIG["L"], H=CONFIG["H"], R=CONFIG["R"], r_c=CONFIG["r_c"],
                    precision=J.PREC_TF32 if args.precision == "tf32" else J.PREC_FP32)
    params = model.synth_params(CONFIG["seed"])
    batches = [J.synth_batch(model, [CONFIG["atoms"]], CONFIG["rho"], CONFIG["seed"] * 100 + m) for m in range(n_mb)]
    cfg["edges_per_structure"] = batches[0].n_edges
    comm = None
    device = local_rank if args.transport == "nccl" else 0
    if N > 1:
        import tempfile

        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if args.transport == "nccl":
            uid = J.Comm.unique_id() if rank == 0 else None
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            comm = J.Comm(obj[0], world, rank, local_rank)
        else:  # all ranks on GPU 0, blocking-rendezvous IPC transport (csrc/transport.hpp)
            obj = [tempfile.mkdtemp(prefix="janus_ipc_") if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            comm = J.Comm.ipc(obj[0], world, rank, 0)
    method_name = args.method or ("wavek" if N > 1 else "symfold")
    method = {"symfold": J.METHOD_SYMFOLD, "wavek": J.METHOD_WAVEK, "onef1b": J.METHOD_ONEF1B}[method_name]
    P = N
    k = min(n_mb, 2 * P)
    max_edges = max(b.n_edges for b in batches) + 64
    tr = J.Trainer(model, params, P, method, n_mb, k=k, max_atoms=CONFIG["atoms"], max_edges=max_edges,
                   max_struct=1, local=(N == 1), graphs=(N == 1), comm=comm, rank=rank, device=device,
                   lanes=(args.lanes if N == 1 else min(args.lanes, 8)))
    for m, b in enumerate(batches):
        tr.load(m, b)
    for _ in range(args.warmup):
        tr.step()

    def barrier():
        if N > 1:
            import torch.distributed as dist
            dist.barrier()

    l2 = []
    times, launches, stats = [], 0, None
    with ClockSampler(device) as clk:
        for _ in range(args.steps):
            flush_l2(l2)
            barrier()
            s = tr.step()
            times.append(s.makespan_ms)
            launches += s.kernel_launches
            stats = s
        # e2e: re-upload every micro-batch from pinned host memory + read the loss back
        pin([a for b in batches for a in (b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target,
                                          b.row_ptr, b.col, b.shift, b.rev)])
        # input-pipelined like a training loop: step k+1's uploads are issued
        # (and queued on the device) while step k runs; every step still copies
        # its own inputs H2D and reads its own loss back D2H (wait()).
        n_e2e = max(5, args.steps)

        def e2e_loop(bs, n=None):
            # two steps in flight: step k+1 is queued on the device before the
            # host reads step k's loss back, so the GPU does not idle on the
            # host between steps; step k+2's uploads and neighbour lists are
            # issued while step k+1 runs
            n = max(2, n or n_e2e)
            barrier()
            t0 = time.perf_counter()
            tr.load_many(bs)
            tr.step_async()
            tr.load_many(bs)
            tr.step_async()
            for _ in range(n - 2):
                tr.wait()
                tr.load_many(bs)
                tr.step_async()
            tr.wait()
            tr.wait()
            return (time.perf_counter() - t0) / n

        # (1) host-built CSR uploaded with the batch (neighbour lists prebuilt
        # once, outside the timed region); (2) device LM: only positions,
        # species, cells and targets cross PCIe and every step rebuilds every
        # micro-batch's neighbour list on the GPU (janus_trainer_load with
        # row_ptr == NULL, nbrlist.cu) — the headline e2e, since a training
        # loop over a dataset must build them per structure
        # untimed: loads alternate between two geometry copies, so the step graph
        # for each parity is captured and instantiated here, outside the timing
        e2e_loop(batches, n=3)
        e2e_host_csr = e2e_loop(batches)
        dev_batches = [J.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target, nl="device")
                       for b in batches]
        tr.load_many(dev_batches)  # untimed: creates the device-LM workspace (pinned + device buffers)
        tr.step()
        e2e_t = [e2e_loop(dev_batches)]
    clocks = clk.summary()
    total_ms = sum(times)
    if N > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
        e = torch.tensor([max(e2e_t)], dtype=torch.float64)
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
        e2e_max = float(e[0])
    else:
        e2e_max = None
    ms_per_step = total_ms / args.steps
    value = n_mb / (ms_per_step / 1000.0)
    e2e_val = n_mb / (e2e_t[0] if e2e_max is None else e2e_max)
    h2d_host_csr = sum(batch_bytes(b) for b in batches)
    # device LM: pos + struct_id to the builder, then the stage block (row_ptr
    # mirror, species, struct_id, pos, cell, targets; row-tile tables not counted)
    h2d = sum(2 * b.pos.nbytes + 2 * b.struct_id.nbytes + b.species.nbytes + b.cell.nbytes + b.E_target.nbytes
              + b.F_target.nbytes + 4 * (b.n_atoms + 1) for b in batches)
    d2h_lm = sum(4 * (b.n_atoms + 1) + 8 for b in batches)  # row_ptr mirror + edge count / status

    # roofline of the dominant edge kernel on the first stage holding a msg unit
    peaks, peak_src = load_peaks()
    roof = None
    if rank == 0:
        try:
            # a block this rank holds (NCCL mode: rank 0 holds only its own blocks)
            st = None
            for blk in ([0] if P == 1 else list(range(P))):
                try:
                    st = tr.stage(blk)
                    break
                except J.JanusError:
                    continue
            if st is None:
                raise J.JanusError(5, "no block held by rank 0")
            # tf32 path: msg_bf_pair_tc (BF weight gradients once per undirected edge pair;
            # the largest edge kernel of the step, profiles/r01_launch_shares_tf32_v14.txt),
            # timed with the step's concurrency: all micro-batches launched on the step's lanes
            # with the step's grid, CUDA events around whole rounds (P == 1; else isolated)
            wk = 4 if args.precision == "tf32" else 2
            if P == 1:  # median of 5 timings of 20 rounds each (single timings vary by up to +-20%)
                runs = sorted((st.time_edge_kernel(wk, -1, iters=20) for _ in range(5)), key=lambda x: x[0])
                ms_bf, ne, fl = runs[2]
                how = ("all micro-batches per round on the step's lanes and grids (CUDA events per round; "
                       "median of 5 x 20 rounds)")
            else:
                ms_bf, ne, fl = st.time_edge_kernel(wk, 0, iters=50)
                how = "one micro-batch, back-to-back launches"
            achieved = fl / (ms_bf * 1e-3) / 1e12
            iso_ms, iso_e, iso_fl = st.time_edge_kernel(wk, 0, iters=50)
            roof = {"kernel": ("msg_bf_pair_tc (tcgen05 kind::f16, bf16 operands, fp32 accumulate; per edge pair)"
                               if args.precision == "tf32" else "msg_bf_kernel (SIMT fp32)"),
                    "bound": "tensor", "achieved": achieved,
                    "peak": peaks["bf16_tflops"], "unit": "TFLOP/s", "frac": achieved / peaks["bf16_tflops"],
                    "traffic": load_traffic(args.precision), "peak_source": f"{peak_src} bf16 dense (MEASURED_PEAKS.json)",
                    "timing": how, "round_ms": ms_bf, "edges_per_round": ne, "flops_per_round": fl,
                    "flops_note": "executed MMA flops: (4RH + 4H^2) x 2 per edge pair = half of that per directed edge",
                    "isolated_launch_ms": iso_ms, "isolated_tflops": iso_fl / (iso_ms * 1e-3) / 1e12,
                    "fp32_simt_nominal_tflops": 74.4}
            fe = st.time_edge_kernel(0, 0, iters=50)
            roof["fe_kernel_tflops"] = fe[2] / (fe[0] * 1e-3) / 1e12
            # step level: executed edge-contraction FLOPs of all four phases (pair mode:
            # once per pair), every layer and micro-batch, over the device-timed step; and
            # the directed-edge algorithm's count (every contraction per directed edge,
            # DESIGN.md §4) over the same time = the rate that algorithm would need
            per_mb = [st.time_edge_kernel(w, 0, iters=5) for w in (0, 1, 2, 3)]
            fl_all = sum(x[2] for x in per_mb)
            if P == 1:
                roof["step_edge_flops"] = fl_all * CONFIG["L"] * n_mb
                roof["step_edge_tflops"] = roof["step_edge_flops"] / (ms_per_step * 1e-3) / 1e12
                roof["step_edge_frac"] = roof["step_edge_tflops"] / peaks["bf16_tflops"]
                e_mb = per_mb[0][1]
                roof["directed_equiv_step_tflops"] = (DIRECTED_FLOP_PER_EDGE * e_mb * CONFIG["L"] * n_mb
                                                      / (ms_per_step * 1e-3) / 1e12)
        except J.JanusError as ex:
            roof = {"error": str(ex)}

    # the fp32 path (north_star tolerances 1e-5 / 1e-4) on the same workload,
    # device-timed the same way: the throughput that meets the tight tolerance,
    # beside the tensor-core headline.  The generic-width path in fp32 (batched
    # per-pair GEMMs, stage_wide.inc) measured 3523 structures/s against the
    # fused fp32 SIMT kernels' 1481, so it is the fp32 path
    fp32_path = None
    if rank == 0 and N == 1 and args.precision == "tf32" and not args.no_fp32_path:
        m32 = J.Model(L=CONFIG["L"], H=CONFIG["H"], R=CONFIG["R"], r_c=CONFIG["r_c"], precision=J.PREC_FP32,
                      generic=True)
        t32 = J.Trainer(m32, params, P, method, n_mb, k=k, max_atoms=CONFIG["atoms"], max_edges=max_edges,
                        max_struct=1, local=True, graphs=True, rank=0, device=local_rank, lanes=args.lanes)
        for m, b in enumerate(batches):
            t32.load(m, b)
        for _ in range(args.warmup):
            t32.step()
        ts32 = []
        for _ in range(min(args.steps, 10)):
            flush_l2(l2)
            ts32.append(t32.step().makespan_ms)
        t32.close()
        ms32 = sum(ts32) / len(ts32)
        fp32_path = {"value": n_mb / (ms32 * 1e-3), "unit": "structures/s", "ms_per_step": ms32, "steps": len(ts32),
                     "dtype": ("fp32-accurate: per-pair products 3xTF32 on tcgen05 (gemm_tc split3), weight-gradient "
                               "and node GEMMs fp32 SIMT (cuBLAS compute type 32F); generic-width path"),
                     "tolerance": "E rel 1e-5, F and gradients 1e-4 of max (tests/test_gpu_bench_parity.py)"}

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        orc = CpuOracle(model_kw, min(os.cpu_count() or 1, n_mb), CONFIG["seed"])
        nthr = len(orc.work)
        v_all, dt_all = orc.run(nthr)
        v_one, dt_one = orc.run(1, per_thread=2)
        cpu = {"value": v_all, "unit": "structures/s", "cores": nthr, "kind": "port",
               "sample": f"{nthr} x 256-atom structures (one per thread), full four-phase step, fp64 oracle "
                         f"(oracle/mlip_oracle.c), {dt_all:.1f} s",
               "one_core": {"value": v_one, "cores": 1, "sample": f"2 x 256-atom structures, {dt_one:.1f} s"}}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "structures/s", "n_gpus": N, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": ("tf32 filters + bf16 BF/BE operands, fp32 accumulate" if args.precision == "tf32"
                         else "fp32"),
               "tolerance": ("E rel 2e-3, F and gradients 2e-2 of max vs the fp64 oracle (tests/test_gpu_bench_parity.py)"
                             if args.precision == "tf32" else "E rel 1e-5, F and gradients 1e-4 of max"),
               "fp32_parity_path": fp32_path,
               "data": "synthetic",
               "config": dict(cfg, precision=args.precision, parallelism=f"pp{P}" if P > 1 else "single-gpu", schedule=method_name,
                              wavek_k=k if method == J.METHOD_WAVEK else None, cuda_graph=(N == 1),
                              lanes=(args.lanes if N == 1 else min(args.lanes, 8)),
                              transport=(None if N == 1 else "nccl (one GPU per rank)" if args.transport == "nccl"
                                         else f"ipc ({N} processes on one GPU)")),
               "e2e": {"value": e2e_val, "unit": "structures/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": 8 * n_mb + d2h_lm, "input_pipelined": True,
                       "neighbour_lists": "rebuilt on the GPU every step (device LM)"},
               "e2e_host_csr": {"value": n_mb / e2e_host_csr, "unit": "structures/s",
                                "h2d_bytes_per_step": h2d_host_csr, "d2h_bytes_per_step": 8 * n_mb,
                                "neighbour_lists": "host-built once, uploaded every step"},
               "gpu_launches": int(launches), "gpu_launches_per_step": int(stats.kernel_launches),
               "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
               "p2p_bytes_per_step": int(stats.p2p_bytes),
               "p2p": ({"GBps_per_gpu": stats.p2p_bytes / (ms_per_step * 1e-3) / 1e9,
                        "nvlink_GBps_per_direction": 900.0,
                        "frac": stats.p2p_bytes / (ms_per_step * 1e-3) / 1e9 / 900.0} if N > 1 else None),
               "loss": stats.loss,
               "peak_hbm_bytes_per_stage": [int(stats.peak_bytes[d]) for d in range(P)]}
        print(json.dumps(out), flush=True)
    tr.close()
    if comm:
        comm.close()


if __name__ == "__main__":
    main()
