#!/usr/bin/env python3
"""configs[2] on one B200: the deep MLIP (L=32, H=256, R=64, r_c=5) on
synthetic 512-atom cells through the generic-width path (stage_wide.inc).

For each run: device-timed structures/s (CUDA events around the step) and the
executor's MEASURED per-device memory: activation slots (live micro-batches,
include/janus/slots.hpp), the pool's bytes and static + arena bytes — SymFold
with the pooled arena vs the same stages with one slot per micro-batch
("unfolded"), and 1F1B-2nd / WaveK for reference, at P = 1 and 8 (P virtual
stages on one GPU, one lane: the pipeline's own order).

Usage: python tools/c3_report.py [--nmb 16] [--prec tf32|fp32] [--out gpurun_out/c3_report.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import paper_2605_18404_b200 as J  # noqa: E402


def run(model, params, batches, P, method, lanes, unfolded=False, k=1, steps=3, warmup=2):
    n = batches[0].n_atoms
    t = J.Trainer(model, params, P, method, len(batches), k=k, max_atoms=n, max_edges=max(b.n_edges for b in batches) + 64,
                  max_struct=1, lanes=lanes, graphs=True, unfolded=unfolded)
    t.load_many(batches)
    for _ in range(warmup):
        t.step(lr=1e-4)
    ms = []
    for _ in range(steps):
        s = t.step(lr=1e-4)
        ms.append(s.makespan_ms)
    ms.sort()
    out = {"P": P, "method": {0: "symfold", 1: "wavek", 2: "onef1b_2nd", 4: "hanayo_2nd"}[method], "k": k,
           "lanes": lanes, "unfolded_slots": unfolded, "ms_per_step": ms[len(ms) // 2],
           "structures_per_s": len(batches) / (ms[len(ms) // 2] / 1e3), "loss": s.loss,
           "kernel_launches": int(s.kernel_launches),
           "memory": [{"device": d, "activation_slots": int(s.act_slots[d]), "activation_pool_bytes": int(s.act_bytes[d]),
                       "static_plus_arena_bytes": int(s.peak_bytes[d])} for d in range(P)]}
    out["peak_hbm_bytes_max_device"] = max(m["static_plus_arena_bytes"] for m in out["memory"])
    t.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nmb", type=int, default=16)
    ap.add_argument("--atoms", type=int, default=512)
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--prec", default="tf32", choices=["tf32", "fp32", "emu"])
    ap.add_argument("--H", type=int, default=256)
    ap.add_argument("--methods", default="all", help="all | symfold (P>1 comparisons off)")
    ap.add_argument("--lanes", type=int, default=8)
    ap.add_argument("--Ps", default="1,8")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c3_report.json"))
    a = ap.parse_args()
    prec = {"tf32": J.PREC_TF32, "fp32": J.PREC_FP32, "emu": J.PREC_FP32_EMU}[a.prec]
    model = J.Model(L=a.L, H=a.H, R=64, precision=prec, generic=True)
    params = model.synth_params(3)
    t0 = time.time()
    batches = [J.synth_batch(model, [a.atoms], 0.095, 900 + m) for m in range(a.nmb)]
    rows = []
    for P in [int(x) for x in a.Ps.split(",")]:
        cases = [(J.METHOD_SYMFOLD, 1, False), (J.METHOD_SYMFOLD, 1, True)]
        if P > 1 and a.methods == "all":
            cases += [(J.METHOD_ONEF1B, 1, False), (J.METHOD_WAVEK, P, False)]
        for method, k, unf in cases:
            lanes = a.lanes if P == 1 else 1
            r = run(model, params, batches, P, method, lanes, unf, k)
            rows.append(r)
            print(json.dumps({x: r[x] for x in ("P", "method", "unfolded_slots", "lanes", "structures_per_s",
                                                "peak_hbm_bytes_max_device")}), flush=True)
    res = {"config": f"L={a.L} H={a.H} R=64 r_c=5, {a.atoms}-atom cells (rho 0.095), N_mb={a.nmb}, "
                     f"{a.prec}, generic-width path, 1 B200 (P virtual stages, 1 lane for P > 1)",
           "edges_per_structure": int(batches[0].n_edges), "wall_s": time.time() - t0, "rows": rows}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
