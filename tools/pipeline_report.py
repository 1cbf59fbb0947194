#!/usr/bin/env python3
"""Pipeline-schedule report on ONE B200: SymFold vs WaveK vs 1F1B-2nd.

All P pipeline stages run in this process on one GPU as virtual devices
(local transport: async device-to-device copies + events), strict device-list
order (lanes = 1), per-instruction CUDA-event timeline.  For each schedule:
  * measured makespan and bubble ratio  sum idle / (P makespan);
  * replay-predicted makespan / bubble of the same schedule under the measured
    mean phase times (graph.hpp:168 replay, the reference's own model);
  * peak live activation bytes per stage from the SPEC lifetime rule
    (FE activations live FE->BE, FF intermediates FF->BF, BF->BE
    injections BF->BE) evaluated on the measured timeline, + static bytes;
  * the executor's MEASURED allocation per device: activation slot pool
    (slots = live micro-batches, include/janus/slots.hpp) and its bytes, next
    to the unfolded arena (one slot per micro-batch) of the same stages.
WaveK's list schedule is generated from the SymFold run's measured phase
means (janus_exec_desc.phase_us), not the paper's ratios.
Virtual devices share the SMs of one GPU, so measured bubbles include
contention; the replay column is the schedule's intrinsic bubble.
Usage: python tools/pipeline_report.py [--out gpurun_out/pipeline_report.json]
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

KIND = {0: "FE", 1: "FF", 2: "BE", 3: "BF"}


def activation_bytes(model, u0, u1, n_atoms):
    """Per-micro-batch bytes of the three lifetime classes for units [u0,u1)."""
    NH4 = n_atoms * model.H * 4
    fe = ff = inj = 0
    for u in range(u0, u1):
        if u == 0:
            fe += NH4
        elif u == model.n_units - 1:
            fe += NH4
            inj += NH4
        elif u % 2 == 1:
            fe += 2 * NH4
            ff += 2 * NH4
            inj += NH4
        else:
            fe += 2 * NH4
            ff += NH4
            inj += NH4
    return fe, ff, inj


def peak_live(tl, dev, sizes):
    """Max over time of live bytes on `dev` from the timeline records."""
    fe_b, ff_b, inj_b = sizes
    ev = []
    by = {}
    for d, k, mb, a, b in tl:
        if int(d) != dev:
            continue
        by.setdefault((int(mb), KIND[int(k)]), []).append((a, b))
    for mb in {m for m, _ in by}:
        def span(kind, pick):
            x = by.get((mb, kind))
            return pick(x) if x else None
        fe0 = span("FE", lambda x: min(a for a, _ in x))
        be1 = span("BE", lambda x: max(b for _, b in x))
        ff0 = span("FF", lambda x: min(a for a, _ in x))
        bf1 = span("BF", lambda x: max(b for _, b in x))
        bf0 = span("BF", lambda x: min(a for a, _ in x))
        if fe0 is not None and be1 is not None:
            ev += [(fe0, fe_b), (be1, -fe_b)]
        elif ff0 is not None and bf1 is not None:  # 1F1B force replica: recomputed FE lives FF->BF
            ev += [(ff0, fe_b), (bf1, -fe_b)]
        if ff0 is not None and bf1 is not None:
            ev += [(ff0, ff_b), (bf1, -ff_b)]
        if bf0 is not None:
            end = be1 if be1 is not None else bf1
            ev += [(bf0, inj_b), (end, -inj_b)]
    live = peak = 0
    for _, x in sorted(ev, key=lambda e: (e[0], e[1])):
        live += x
        peak = max(peak, live)
    return peak


def run(model, params, batches, P, method, k, steps=3, warmup=2, phase_us=None):
    kw = dict(k=k, max_atoms=batches[0].n_atoms, max_edges=max(b.n_edges for b in batches) + 64, max_struct=1,
              lanes=1, phase_us=phase_us)
    t = J.Trainer(model, params, P, method, len(batches), timeline=True, **kw)
    for i, b in enumerate(batches):
        t.load(i, b)
    for _ in range(warmup):
        t.step()
    stats, tls = [], []
    for _ in range(steps):
        stats.append(t.step())
        tls.append(t.timeline())
    i = int(np.argsort([s.makespan_ms for s in stats])[len(stats) // 2])
    s, tl = stats[i], tls[i]
    phase = {}
    for name, kk in (("FE", 0), ("FF", 1), ("BE", 2), ("BF", 3)):
        d = tl[tl[:, 1] == kk]
        phase[name] = float((d[:, 4] - d[:, 3]).mean()) if len(d) else 0.0
    text = t.schedule_text()
    # replay with measured per-instruction means (FF of 1F1B already contains the recompute)
    ff = phase["FF"] - (phase["FE"] if method in (J.METHOD_ONEF1B, J.METHOD_HANAYO) else 0.0)
    pred_ms, pred_bubble = J.schedule_replay(text, phase["FE"], max(ff, 1e-6), phase["BE"], phase["BF"])
    plan = t.plan()
    mem = []
    for dv in range(P):
        blocks = [b for b in range(P) if J_device_of(text, b, P, "E") == dv] + \
                 [b for b in range(P) if J_device_of(text, b, P, "F") == dv]
        sizes = [0, 0, 0]
        for b in sorted(set(blocks)):  # every block whose stage object lives on this device
            for q, x in enumerate(activation_bytes(model, int(plan[b][0]), int(plan[b][1]), batches[0].n_atoms)):
                sizes[q] += x
        peak = peak_live(tl, dv, sizes)
        mem.append({"device": dv, "static_plus_arena_bytes": int(s.peak_bytes[dv]), "peak_live_activation_bytes": int(peak),
                    "activation_slots": int(s.act_slots[dv]), "activation_pool_bytes": int(s.act_bytes[dv])})
    # the unfolded arena (one slot per micro-batch) of the same stages, for comparison
    tu = J.Trainer(model, params, P, method, len(batches), unfolded=True, **kw)
    for i, b in enumerate(batches):
        tu.load(i, b)
    su = tu.step()
    tu.close()
    for dv in range(P):
        mem[dv]["unfolded_pool_bytes"] = int(su.act_bytes[dv])
        mem[dv]["unfolded_static_plus_arena_bytes"] = int(su.peak_bytes[dv])
    out = {"P": P, "method": {0: "symfold", 1: "wavek", 2: "onef1b_2nd", 4: "hanayo_2nd"}[method], "k": k,
           "wavek_phase_us": list(phase_us) if phase_us else None,
           "peak_hbm_bytes_max_device": max(m["static_plus_arena_bytes"] for m in mem),
           "makespan_ms": s.makespan_ms, "structures_per_s": len(batches) / (s.makespan_ms / 1e3),
           "bubble_measured": s.bubble_ratio, "busy_ms": [s.busy_ms[d] for d in range(P)],
           "phase_mean_us": {k2: v * 1e3 / 1e3 for k2, v in phase.items()},
           "replay_makespan_ms": pred_ms / 1e3, "bubble_replay": pred_bubble,
           "p2p_bytes_per_step": int(s.p2p_bytes), "memory": mem,
           "timeline_ascii": J.render_timeline(recs=tl, quantum=max(s.makespan_ms * 1e3 / 160, 1e-3))}
    t.close()
    return out


def J_device_of(text, block, P, side):
    """Device of energy (vs=block) or force (vs=2P-1-block) stage from the schedule text."""
    vs = block if side == "E" else 2 * P - 1 - block
    for line in text.splitlines()[1:]:
        f = line.split()
        if f[2] in ("FE", "FF", "BE", "BF") and f[4] == f"vs={vs}":
            return int(f[0][1:])
    return -1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "pipeline_report.json"))
    ap.add_argument("--Ps", default="2,4,8")
    ap.add_argument("--nmb", type=int, default=32)
    ap.add_argument("--kmult", default="0.5,1,2,4",
                    help="WaveK candidate unit sizes k = m P (divisors of N_mb only): the paper's offline sweep "
                         "(PAPER.md:865, 'evaluate a few candidate k values ... and select the best')")
    args = ap.parse_args()
    model = J.Model(L=4, H=64, R=64, precision=J.PREC_TF32)
    params = model.synth_params(7)
    batches = [J.synth_batch(model, [256], 0.095, 700 + m) for m in range(args.nmb)]
    rows = []
    for P in [int(x) for x in args.Ps.split(",")]:
        ph = None
        ks = sorted({max(1, int(round(float(f) * P))) for f in args.kmult.split(",")})
        ks = [k for k in ks if k <= args.nmb and args.nmb % k == 0]
        cases = [(J.METHOD_SYMFOLD, 1), (J.METHOD_ONEF1B, 1), (J.METHOD_HANAYO, 1)] + [(J.METHOD_WAVEK, k) for k in ks]
        for method, k in cases:
            r = run(model, params, batches, P, method, k, phase_us=ph if method == J.METHOD_WAVEK else None)
            if method == J.METHOD_SYMFOLD:  # WaveK's cost model: this box's measured phase means
                m = r["phase_mean_us"]
                ph = (m["FE"], m["FF"], m["BE"], m["BF"])
            rows.append(r)
            print(json.dumps({x: r[x] for x in ("P", "method", "k", "makespan_ms", "structures_per_s", "bubble_measured",
                                                "bubble_replay", "peak_hbm_bytes_max_device")}), flush=True)
    summary = []
    for P in sorted({r["P"] for r in rows}):
        sf = next(r for r in rows if r["P"] == P and r["method"] == "symfold")
        wk = max((r for r in rows if r["P"] == P and r["method"] == "wavek"), key=lambda r: r["structures_per_s"])
        summary.append({"P": P, "symfold": sf["structures_per_s"], "wavek_best_k": wk["k"],
                        "wavek_best": wk["structures_per_s"], "wavek_over_symfold": wk["structures_per_s"] / sf["structures_per_s"],
                        "bubble_symfold": sf["bubble_measured"], "bubble_wavek_best": wk["bubble_measured"]})
        print(json.dumps(summary[-1]), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"config": "C2: L=4 H=64 R=64, 256-atom cells, N_mb=%d, tf32, 1 GPU, lanes=1" % args.nmb, "rows": rows,
               "wavek_sweep": summary}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
