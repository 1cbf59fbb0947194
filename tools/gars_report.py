#!/usr/bin/env python3
"""GARS on the device step (configs[3]-style mixed cells, one B200).

A global batch of M periodic cells with sizes drawn from the C4 set
{128, 250, 256, 432, 500, 512, 686, 864, 1000, 1024} is
split into N_mb micro-batches twice — GARS pack-and-shuffle (janus_gars_pack)
and the greedy sequential fixed-atom baseline (janus_gars_greedy, PAPER.md:
917-918) — from the SAME cells (positions seeded per graph id).  Each packing
trains through the trainer on a P-stage SymFold pipeline (virtual stages on
one GPU, strict list order, per-instruction timeline) with device-built
neighbour lists, and we report per-micro-batch atom std, measured makespan,
atoms/s and bubble ratio.  Usage: python tools/gars_report.py [--P 4]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_18404_b200 as J  # noqa: E402

C4_SIZES = [128, 250, 256, 432, 500, 512, 686, 864, 1000, 1024]


def build_batches(model, cells, groups):
    out = []
    for g in groups:
        P, S, SID, C, E, F = [], [], [], [], [], []
        for s, gid in enumerate(g):
            pos, sp, L, Et, Ft = cells[gid]
            P.append(pos); S.append(sp); SID.append(np.full(len(pos), s, np.int32)); C.append(L)
            E.append(Et); F.append(Ft)
        out.append(J.Batch(np.concatenate(P), np.concatenate(S), np.concatenate(SID), np.array(C), np.array(E),
                           np.concatenate(F), nl="device"))
    return out


def run(model, params, batches, P, steps, lanes):
    max_atoms = max(b.n_atoms for b in batches)
    max_struct = max(b.n_struct for b in batches)
    tr = J.Trainer(model, params, P, J.METHOD_SYMFOLD, len(batches), max_atoms=max_atoms,
                   max_edges=max_atoms * 64, max_struct=max_struct, graphs=False, timeline=(lanes == 1),
                   lanes=lanes)
    tr.load_many(batches)
    tr.step()
    ms, bub = [], []
    for _ in range(steps):
        s = tr.step()
        ms.append(s.makespan_ms)
        bub.append(s.bubble_ratio)
    tr.close()
    return statistics.median(ms), statistics.median(bub)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=4)
    ap.add_argument("--M", type=int, default=64, help="structures per global batch")
    ap.add_argument("--n-mb", type=int, default=16)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=11)
    args = ap.parse_args()
    model = J.Model(L=4, H=64, R=64, r_c=5.0, precision=J.PREC_TF32)
    params = model.synth_params(7)
    rng = np.random.default_rng(args.seed)
    sizes = [int(x) for x in rng.choice(C4_SIZES, size=args.M)]
    cells = [J.synth_cell(n, 0.095, model.n_species, 50000 + i) for i, n in enumerate(sizes)]
    total = sum(sizes)
    res = {"config": f"configs[3]-style: {args.M} cells of {sorted(set(sizes))} atoms, N_mb={args.n_mb}, "
                     f"L=4 H=64, tf32, SymFold P={args.P} (virtual stages on one GPU)", "total_atoms": total}
    for name, greedy in (("gars", False), ("greedy_sequential", True)):
        packing = J.gars_pack(sizes, args.n_mb, 1, seed=args.seed, greedy=greedy)
        groups = [g for g, _ in packing]
        tot = [sum(sizes[i] for i in g) for g in groups]
        batches = build_batches(model, cells, groups)
        ms_p, bub = run(model, params, batches, args.P, args.steps, lanes=1)
        ms_1, _ = run(model, params, batches, 1, args.steps, lanes=8)
        res[name] = {"mb_atoms_std": float(np.std(tot)), "mb_atoms_max": int(max(tot)), "mb_atoms_min": int(min(tot)),
                     f"P{args.P}_makespan_ms": ms_p, f"P{args.P}_atoms_per_s": total / (ms_p * 1e-3),
                     f"P{args.P}_bubble_ratio": bub, "P1_lanes8_makespan_ms": ms_1,
                     "P1_lanes8_atoms_per_s": total / (ms_1 * 1e-3)}
        print(name, json.dumps(res[name]), flush=True)
    g, q = res["gars"], res["greedy_sequential"]
    res["speedup_gars_over_greedy"] = {f"P{args.P}": q[f"P{args.P}_makespan_ms"] / g[f"P{args.P}_makespan_ms"],
                                       "P1": q["P1_lanes8_makespan_ms"] / g["P1_lanes8_makespan_ms"]}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
