#!/usr/bin/env python3
"""Throughput of the four-phase step on the BASELINE.json configs that fit the
H=64 kernels, one B200, device-timed (CUDA graph, L2 flushed between steps),
tf32 tensor-core path, device-built neighbour lists:

  C1  L=4 H=64, 64-atom cells, 4 micro-batches (the CPU reference's case)
  C2  L=4 H=64, 256-atom cells, 32 micro-batches (bench.py's workload)
  C4  L=4 H=64, mixed 128..1024-atom cells packed by GARS into 16 micro-batches
  C5  L=4 H=64, 4096-atom cells at rho 0.19 (~100 neighbours), 8 micro-batches

(C3, H=256, runs on the generic-width path: tools/c3_report.py.)  One JSON
line per config: structures/s, atoms/s, edges/s and step-level edge TFLOP/s.
"""
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2605_18404_b200 as J  # noqa: E402
from bench import flush_l2  # noqa: E402
from gars_report import C4_SIZES, build_batches  # noqa: E402

FLOP_PER_EDGE = 2.0 * ((64 * 64 + 64 * 64) + (2 * 64 * 64 + 2 * 64 * 64 + 64) + (4 * 64 * 64 + 6 * 64 * 64) +
                       (2 * 64 * 64 + 3 * 64 * 64))  # FE + FF + BF + BE per layer (stage.cu edge_kernel_flops_per_edge)


def measure(name, model, params, batches, lanes=None, steps=10, warmup=3):
    lanes = lanes or len(batches)  # one lane per micro-batch, as bench.py
    na = max(b.n_atoms for b in batches)
    t = J.Trainer(model, params, 1, J.METHOD_SYMFOLD, len(batches), max_atoms=na, max_edges=na * 140,
                  max_struct=max(b.n_struct for b in batches), graphs=True, lanes=lanes)
    t.load_many(batches)
    for _ in range(warmup):
        t.step()
    l2, ms = [], []
    for _ in range(steps):
        flush_l2(l2)
        ms.append(t.step().makespan_ms)
    # edge counts from the stage geometry are not exported; rebuild on the host for the count
    E = sum(int(J.nbrlist_device(b.pos, b.struct_id, b.cell, model.r_c, max_edges=b.n_atoms * 140)[0][-1])
            for b in batches)
    t.close()
    m = statistics.median(ms)
    S = sum(b.n_struct for b in batches)
    A = sum(b.n_atoms for b in batches)
    out = {"config": name, "ms_per_step": m, "structures_per_s": S / (m * 1e-3), "atoms_per_s": A / (m * 1e-3),
           "edges_per_step": E, "step_edge_tflops": FLOP_PER_EDGE * model.L * E / (m * 1e-3) / 1e12,
           "lanes": lanes, "n_micro_batches": len(batches)}
    print(json.dumps(out), flush=True)
    return out


def main():
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    # --fp32: the generic-width fp32 path (bench.py's fp32_parity_path); --steps / --warmup: shorter runs (ncu)
    kw = {}
    if "--steps" in sys.argv:
        kw["steps"] = int(sys.argv[sys.argv.index("--steps") + 1])
    if "--warmup" in sys.argv:
        kw["warmup"] = int(sys.argv[sys.argv.index("--warmup") + 1])
    if "--fp32" in sys.argv:
        model = J.Model(L=4, H=64, R=64, r_c=5.0, precision=J.PREC_FP32, generic=True)
    elif "--generic" in sys.argv:  # the generic-width path in tf32 (configs[2]'s path) on these configs
        model = J.Model(L=4, H=64, R=64, r_c=5.0, precision=J.PREC_TF32, generic=True)
    else:
        model = J.Model(L=4, H=64, R=64, r_c=5.0, precision=J.PREC_TF32)
    params = model.synth_params(7)
    if only in (None, "C1"):
        measure("C1: 64-atom cells, N_mb=4", model, params,
                [J.synth_batch(model, [64], 0.095, 10 + i, device_nl=True) for i in range(4)], **kw)
    if only in (None, "C2"):
        measure("C2: 256-atom cells, N_mb=32", model, params,
                [J.synth_batch(model, [256], 0.095, 700 + i, device_nl=True) for i in range(32)], **kw)
    if only is not None:
        return
    rng = np.random.default_rng(11)
    sizes = [int(x) for x in rng.choice(C4_SIZES, size=64)]
    cells = [J.synth_cell(n, 0.095, model.n_species, 50000 + i) for i, n in enumerate(sizes)]
    groups = [g for g, _ in J.gars_pack(sizes, 16, 1, seed=11)]
    measure("C4: 64 mixed 128..1024-atom cells, GARS -> N_mb=16", model, params, build_batches(model, cells, groups))
    measure("C5: 4096-atom cells rho=0.19, N_mb=8", model, params,
            [J.synth_batch(model, [4096], 0.19, 4000 + i, device_nl=True) for i in range(8)])


if __name__ == "__main__":
    main()
