import os, sys, time
sys.path.insert(0, os.getcwd())
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
bench.pin([a for b in batches for a in (b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target, b.row_ptr, b.col, b.shift, b.rev)])
for rep in range(4):
    t0 = time.perf_counter(); tr.step_async(); t1 = time.perf_counter()
    for m, b in enumerate(batches): tr.load(m, b)
    t2 = time.perf_counter(); s = tr.wait(); t3 = time.perf_counter()
    print(f"step_async {1e3*(t1-t0):.3f}  loads {1e3*(t2-t1):.3f}  wait {1e3*(t3-t2):.3f}  dev {s.makespan_ms:.3f}", flush=True)
import ctypes
hb = batches[0].c()
t0 = time.perf_counter()
for _ in range(100): J.check(J._lib.janus_trainer_load(tr.h, 0, ctypes.byref(hb)))
t1 = time.perf_counter()
for _ in range(100): hb = batches[0].c()
t2 = time.perf_counter()
print(f"C load {1e6*(t1-t0)/100:.1f} us, python struct {1e6*(t2-t1)/100:.1f} us")
