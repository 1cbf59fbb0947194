#!/usr/bin/env python3
"""Where the end-to-end loop's time goes (C2, device LM every step): host
wall time of each call of bench.py's e2e loop (load_many / step_async /
wait) against the device step time, to tell a host-bound loop from a
device-bound one.  Usage: python tools/e2e_probe.py [--steps 30]"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import paper_2605_18404_b200 as J  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    a = ap.parse_args()
    m = J.Model(L=4, H=64, R=64, r_c=5.0, precision=J.PREC_TF32)
    params = m.synth_params(7)
    bs = [J.synth_batch(m, [256], 0.095, 700 + i) for i in range(32)]
    dev = [J.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target, nl="device") for b in bs]
    tr = J.Trainer(m, params, 1, J.METHOD_SYMFOLD, 32, max_atoms=256, max_edges=max(b.n_edges for b in bs) + 64,
                   max_struct=1, graphs=True, lanes=32)
    for _ in range(4):
        tr.load_many(dev)
        tr.step()
    tl, ts, tw, dev_ms = [], [], [], []
    tr.load_many(dev)
    tr.step_async()
    t_start = time.perf_counter()
    for _ in range(a.steps):
        t0 = time.perf_counter()
        tr.load_many(dev)
        t1 = time.perf_counter()
        tr.step_async()
        t2 = time.perf_counter()
        s = tr.wait()
        t3 = time.perf_counter()
        tl.append(t1 - t0)
        ts.append(t2 - t1)
        tw.append(t3 - t2)
        dev_ms.append(s.makespan_ms)
    total = time.perf_counter() - t_start
    tr.wait()
    med = lambda x: 1e3 * statistics.median(x)  # noqa: E731
    out = {"steps": a.steps, "e2e_ms_per_step": 1e3 * total / a.steps, "host_load_many_ms": med(tl),
           "host_step_async_ms": med(ts), "host_wait_ms": med(tw), "device_step_ms": statistics.median(dev_ms)}
    print(json.dumps(out))
    tr.close()


if __name__ == "__main__":
    main()
