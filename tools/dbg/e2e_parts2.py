"""Where does the e2e loop lose time vs the device-timed step? (C2 bench config)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_18404_b200 as J
m = J.Model(L=4, H=64, R=64, precision=J.PREC_TF32)
params = m.synth_params(7)
host = [J.synth_batch(m, [256], 0.095, 700 + i) for i in range(32)]
dev = [J.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target, nl="device") for b in host]
tr = J.Trainer(m, params, 1, J.METHOD_SYMFOLD, 32, max_atoms=256, max_edges=14000, max_struct=1, graphs=True, lanes=16)
tr.load_many(dev); tr.step(); tr.load_many(host); tr.step()
def loop(bs, n=20, load=True):
    t0 = time.perf_counter()
    if load: tr.load_many(bs)
    tr.step_async()
    tl = 0.0
    for _ in range(n - 1):
        a = time.perf_counter()
        if load: tr.load_many(bs)
        tl += time.perf_counter() - a
        tr.wait(); tr.step_async()
    s = tr.wait()
    return (time.perf_counter() - t0) / n * 1e3, tl / (n - 1) * 1e3, s.makespan_ms
for name, bs, ld in (("no loads", host, False), ("host CSR", host, True), ("device LM", dev, True)):
    for _ in range(2):
        ms, lms, dev_ms = loop(bs, load=ld)
    print(f"{name:10s} e2e {ms:.3f} ms/step  host load_many {lms:.3f} ms  device step {dev_ms:.3f} ms", flush=True)
