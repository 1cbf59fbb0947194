"""The BENCHMARKED step pinned to the fp64 oracle.

bench.py's exact configuration — L=4, H=R=64, r_c=5, 256-atom fcc cells at
rho=0.095 with the bench's seeds, SymFold P=1 in pair mode, 32 compute lanes
(which fix the tiles per CTA and so the BF/BE partial grouping), device-built
neighbour lists (device LM) and CUDA-graph replay — run through the trainer
API on two of the bench's micro-batches, and compared per micro-batch with
oracle.step on the same inputs:

* tensor-core mode (tf32 filters + bf16 BF/BE operands, fp32 accumulate):
  E relative 5e-3, F and gradients 2e-2 of the max magnitude (measured on
  the bench config: E 1e-4, F 2.5e-3, g 5e-4, g2 3.6e-3; the mixed C4 cells
  reach E 2.2e-3: a 1024-atom energy sums 1024 tf32-filtered atom terms);
* fp32 SIMT parity mode: E relative 1e-5, F and gradients 1e-4 (north_star).

Also here: the step's loss and the Adam update (OS) against the oracle, a
mixed-size C4 micro-batch (128..1024-atom cells) and a C5 4096-atom dense
cell at L=1 against the oracle.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"tf32": (5e-3, 2e-2, 2e-2), "fp32": (1e-5, 1e-4, 1e-4)}
BENCH = dict(L=4, H=64, R=64, r_c=5.0, atoms=256, rho=0.095, seed=7)


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


def oracle_steps(oracle, m, batches, params):
    om = oracle.Model(L=m.L, H=m.H, R=m.R, n_species=m.n_species, r_c=m.r_c, w_E=m.w_E, w_F=m.w_F)

    def one(b):
        ob = oracle.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target.astype(float), b.F_target.astype(float))
        return oracle.step(om, ob, oracle.build_nbrlist(om, ob), params.astype(np.float64))

    with ThreadPoolExecutor(max_workers=len(batches)) as ex:
        return list(ex.map(one, batches))


def run_trainer(janus, m, params, batches, lanes, lr=1e-3, steps=1, max_atoms=None, max_struct=1):
    n_mb = len(batches)
    max_atoms = max_atoms or max(b.n_atoms for b in batches)
    tr = janus.Trainer(m, params, 1, janus.METHOD_SYMFOLD, n_mb, max_atoms=max_atoms,
                       max_edges=max(b.n_edges for b in batches) + 64,
                       max_struct=max_struct, local=True, graphs=True, lanes=lanes)
    dev = [janus.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target, nl="device") for b in batches]
    stats = []
    for _ in range(steps):
        tr.load_many(dev)  # device LM, as bench.py's e2e
        stats.append(tr.step(lr=lr))
    return tr, stats


def compare(janus, m, tr, batches, refs, prec, tag):
    tol_e, tol_f, tol_g = TOL[prec]
    st = tr.stage(0)
    worst = {}
    for mb, (b, r) in enumerate(zip(batches, refs)):
        E, _ = st.energy(mb, b.n_struct)
        F, _ = st.forces(mb, b.n_atoms)
        errs = dict(E=rel(E, r.E), F=rel(F, r.F), g1=rel(st.grads(1, mb), r.grad1), g2=rel(st.grads(2, mb), r.grad2),
                    g=rel(st.grads(0, mb), r.grad))
        for k, v in errs.items():
            worst[k] = max(worst.get(k, 0.0), v)
    print(f"{tag} [{prec}] worst relative errors vs the fp64 oracle: {worst}")
    assert worst["E"] < tol_e and worst["F"] < tol_f
    assert worst["g1"] < tol_g and worst["g2"] < tol_g and worst["g"] < tol_g
    return worst


@pytest.fixture(scope="module")
def bench_case(janus, oracle, has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")
    m = janus.Model(L=BENCH["L"], H=BENCH["H"], R=BENCH["R"], r_c=BENCH["r_c"])
    params = m.synth_params(BENCH["seed"])
    # micro-batches 0 and 1 of bench.py (seed * 100 + m)
    batches = [janus.synth_batch(m, [BENCH["atoms"]], BENCH["rho"], BENCH["seed"] * 100 + mb) for mb in range(2)]
    refs = oracle_steps(oracle, m, batches, params)
    return m, params, batches, refs


@pytest.mark.parametrize("prec,generic", [("tf32", False), ("fp32", False), ("fp32", True)])
def test_bench_config_matches_oracle(janus, oracle, bench_case, prec, generic):
    """generic: the fp32 path bench.py reports beside the headline (the
    generic-width GEMM path, stage_wide.inc) at the fp32 tolerances."""
    m0, params, batches, refs = bench_case
    m = janus.Model(L=m0.L, H=m0.H, R=m0.R, r_c=m0.r_c,
                    precision=janus.PREC_TF32 if prec == "tf32" else janus.PREC_FP32, generic=generic)
    lr = 1e-3
    tr, stats = run_trainer(janus, m, params, batches, lanes=32, lr=lr)
    compare(janus, m, tr, batches, refs, prec, "bench config (L=4, 256-atom fcc, 32 lanes, device LM, graphs)")
    # the printed loss (sum over micro-batches of L_E + L_F) and the OS update
    loss_ref = sum(r.loss for r in refs)
    assert abs(stats[0].loss - loss_ref) < (2e-3 if prec == "tf32" else 1e-5) * abs(loss_ref)
    g = sum(r.grad for r in refs)
    p, m1, m2 = params.astype(np.float64).copy(), np.zeros(g.size), np.zeros(g.size)
    oracle.adam(p, m1, m2, g, lr, 0.9, 0.999, 1e-8, 1)
    p_gpu = tr.params()
    # Adam's first step moves each parameter by ~lr * sign(g): compare the update
    d_ref, d_gpu = p - params, p_gpu.astype(np.float64) - params
    ok = np.abs(g) > (5e-2 if prec == "tf32" else 1e-3) * np.abs(g).max()  # sign-stable entries
    frac = float(np.mean(np.abs(d_gpu[ok] - d_ref[ok]) < 1e-2 * lr))
    print(f"Adam update agreement ({prec}): {frac:.5f} of {ok.sum()} sign-stable entries")
    assert frac > (0.99 if prec == "tf32" else 0.999)
    tr.close()


def test_bench_config_graph_replay_stable(janus, bench_case):
    """Two more replayed steps on re-loaded inputs (the two geometry parities
    alternate, so both cached graphs run): the loss tracks the first step's
    loss trend and stays finite, and replays at a CHANGED learning rate use the
    new value (the optimizer reads its hyperparameters on the device)."""
    m0, params, batches, _ = bench_case
    m = janus.Model(L=m0.L, H=m0.H, R=m0.R, r_c=m0.r_c, precision=janus.PREC_TF32)
    tr, st = run_trainer(janus, m, params, batches, lanes=32, lr=1e-3, steps=3)
    assert all(np.isfinite(s.loss) for s in st)
    p_before = tr.params()
    tr.load_many([janus.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target, b.F_target, nl="device")
                  for b in batches])
    tr.step(lr=0.0)  # same geometry parity as an earlier captured graph: replayed with lr = 0
    assert np.array_equal(tr.params(), p_before)
    tr.close()


@pytest.mark.parametrize("prec,generic", [("tf32", False), ("fp32", False), ("fp32", True)])
def test_c4_mixed_cells_match_oracle(janus, oracle, has_gpu, prec, generic):
    """configs[3]'s mixed 128-1024-atom cells, two per micro-batch."""
    if not has_gpu:
        pytest.skip("no GPU")
    m = janus.Model(L=4, H=64, R=64, precision=janus.PREC_TF32 if prec == "tf32" else janus.PREC_FP32, generic=generic)
    params = m.synth_params(8)
    batches = [janus.synth_batch(m, [128, 1024], 0.095, 31), janus.synth_batch(m, [686, 250], 0.095, 32)]
    refs = oracle_steps(oracle, m, batches, params)
    tr, _ = run_trainer(janus, m, params, batches, lanes=8, max_atoms=1152, max_struct=2)
    compare(janus, m, tr, batches, refs, prec, "C4 mixed cells")
    tr.close()


def test_c5_dense_cell_matches_oracle(janus, oracle, has_gpu):
    """configs[4]: a 4096-atom cell at rho=0.19 (~100 neighbours/atom), L=1,
    tensor-core mode, against the oracle."""
    if not has_gpu:
        pytest.skip("no GPU")
    m = janus.Model(L=1, H=64, R=64, precision=janus.PREC_TF32)
    params = m.synth_params(9)
    batches = [janus.synth_batch(m, [4096], 0.19, 41)]
    refs = oracle_steps(oracle, m, batches, params)
    tr, _ = run_trainer(janus, m, params, batches, lanes=1)
    compare(janus, m, tr, batches, refs, "tf32", "C5 4096-atom dense cell")
    tr.close()
