#!/usr/bin/env python3
"""Step time vs number of micro-batches (one lane each) on the C2 cell: the
1-micro-batch time is the chain latency; the slope is the throughput cost."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2605_18404_b200 as J  # noqa: E402
from bench import flush_l2  # noqa: E402

model = J.Model(L=4, H=64, R=64, r_c=5.0, precision=J.PREC_TF32)
params = model.synth_params(7)
allb = [J.synth_batch(model, [256], 0.095, 700 + i, device_nl=True) for i in range(32)]
for n in (1, 2, 4, 8, 16, 32):
    t = J.Trainer(model, params, 1, J.METHOD_SYMFOLD, n, max_atoms=256, max_edges=256 * 140, max_struct=1,
                  graphs=True, lanes=n)
    t.load_many(allb[:n])
    for _ in range(3):
        t.step()
    l2, ms = [], []
    for _ in range(10):
        flush_l2(l2)
        ms.append(t.step().makespan_ms)
    t.close()
    m = statistics.median(ms)
    print(f"n_mb={n:2d} ms_per_step={m:.3f} structures/s={n / m * 1e3:.0f}", flush=True)
