import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
import paper_2605_18404_b200 as J
cfg = bench.CONFIG
model = J.Model(L=cfg["L"], H=cfg["H"], R=cfg["R"], r_c=cfg["r_c"], precision=J.PREC_TF32)
params = model.synth_params(cfg["seed"])
batches = [J.synth_batch(model, [cfg["atoms"]], cfg["rho"], cfg["seed"] + 1 + m) for m in range(cfg["n_mb"])]
tr = J.Trainer(model, params, 1, J.METHOD_SYMFOLD, cfg["n_mb"], k=2, max_atoms=cfg["atoms"], max_edges=max(b.n_edges for b in batches) + 64,
               max_struct=1, local=True, graphs=True, lanes=16)
for m, b in enumerate(batches): tr.load(m, b)
for _ in range(3): tr.step()
bench.pin([a for b in batches for a in (b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target, b.row_ptr, b.col, b.shift, b.rev)]) if hasattr(bench, "pin") else None
for rep in range(3):
    t0 = time.perf_counter()
    for m, b in enumerate(batches): tr.load(m, b)
    t1 = time.perf_counter()
    s = tr.step()
    t2 = time.perf_counter()
    print(f"load {1e3*(t1-t0):.2f} ms  step(host) {1e3*(t2-t1):.2f} ms  step(dev) {s.makespan_ms:.2f} ms", flush=True)
