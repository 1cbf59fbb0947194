#!/usr/bin/env python3
"""configs[2] memory study (deep MLIP L=32, H=256, 512-atom cells, P=8):
SymFold vs the unfolded 1F1B-2nd baseline, peak bytes per stage by the SPEC
lifetime rule (include/janus/tuner.hpp peak_memory) on the
replayed schedules.  MODEL-BASED: the H=256 edge kernels are not built
(DESIGN.md §7), so activation bytes come from the stage arena's lifetime
classes at H=256 (the executor's own per-unit buffers, tools/pipeline_report
activation_bytes) and static bytes from the parameter counts (params, grads,
Adam m1/m2, transposed copies, two per-micro-batch gradient ledgers).
Phase times: Table 4 UMA-1.2B ratios (only the overlap pattern matters).
Host only: python tools/c3_memory_report.py [--nmb 16]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2605_18404_b200 as J  # noqa: E402
from pipeline_report import activation_bytes  # noqa: E402

UMA = (26.25, 37.51, 43.59, 82.03)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nmb", type=int, default=16)
    ap.add_argument("--P", type=int, default=8)
    args = ap.parse_args()
    P, N, atoms = args.P, args.nmb, 512
    m = J.Model(L=32, H=256, R=64)
    plan = J.plan_stages(m, P)
    fe = ff = 0
    static = []
    for b in range(P):
        u0, u1 = int(plan[b][0]), int(plan[b][1])
        a, f, inj = activation_bytes(m, u0, u1, atoms)
        fe, ff = max(fe, a + inj), max(ff, f)
        n_par = (m.unit_offset(u1) if u1 < m.n_units else m.param_count()) - m.unit_offset(u0)
        static.append(4.0 * n_par * (4 + 1 + 2 * N))  # params, grad, m1, m2, transposes, g1/g2 ledgers
    out = {"config": f"configs[2]: L=32 H=256 R=64, {atoms}-atom cells, P={P}, N_mb={N} (cost model, lifetime rule)",
           "fe_bytes_per_mb": fe, "ff_bytes_per_mb": ff, "static_bytes_per_stage": static}
    for name, meth in (("symfold", J.METHOD_SYMFOLD), ("onef1b_2nd_unfolded", J.METHOD_ONEF1B),
                       ("hanayo_2nd", J.METHOD_HANAYO), ("wavek_k2P", J.METHOD_WAVEK)):
        text = J.schedule_text(meth, P, N, 2 * P)
        if meth == J.METHOD_ONEF1B:
            # linear map floor(s_v/2): energy device d < P/2 holds blocks 2d, 2d+1; force device
            # P/2 + d' holds the replicas of blocks P-1-2d', P-2-2d' (full params + Adam state)
            st = [static[2 * d] + static[2 * d + 1] if d < P // 2 else
                  static[P - 1 - 2 * (d - P // 2)] + static[P - 2 - 2 * (d - P // 2)] for d in range(P)]
            # each device keeps the activations of its TWO virtual stages
            peaks = J.schedule_memory(text, UMA, st, fe, ff, replicate=False)
        else:
            peaks = J.schedule_memory(text, UMA, static, fe, ff, replicate=False)
        ms, bub = J.schedule_replay(text, *UMA)
        out[name] = {"peak_bytes_per_device": [float(x) for x in peaks], "max_peak_GB": float(max(peaks)) / 1e9,
                     "replay_makespan": ms, "replay_bubble": bub}
        print(name, f"max peak {max(peaks) / 1e9:.2f} GB", [round(x / 1e9, 2) for x in peaks], flush=True)
    out["symfold_over_unfolded_max_peak"] = out["symfold"]["max_peak_GB"] / out["onef1b_2nd_unfolded"]["max_peak_GB"]
    print(json.dumps({k: out[k] for k in ("config", "symfold_over_unfolded_max_peak")}))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "r01_c3_memory_model.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
