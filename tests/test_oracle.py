"""The fp64 oracle is pinned before it is trusted: PyTorch fp64 autograd
double-backward goldens (tests/golden/mlip_golden.npz), central finite
differences, and the Eq. (2) ledger identity."""
import os

import numpy as np
import pytest

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mlip_golden.npz"))
CASES = sorted({k.split("__")[0] for k in GOLD.files})


def load_case(O, name):
    g = {k.split("__")[1]: GOLD[k] for k in GOLD.files if k.startswith(name + "__")}
    L, H, R, S = map(int, g["model"])
    rc, wE, wF = map(float, g["model_f"])
    model = O.Model(L=L, H=H, R=R, n_species=S, r_c=rc, w_E=wE, w_F=wF)
    batch = O.Batch(g["pos"], g["species"], g["struct_id"], g["cell"], g["E_target"], g["F_target"])
    return model, batch, g


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_autograd_golden(oracle, name):
    model, batch, g = load_case(oracle, name)
    nl = oracle.build_nbrlist(model, batch)
    # integer work is bit-exact
    assert np.array_equal(nl.row_ptr, g["row_ptr"]) and np.array_equal(nl.col, g["col"])
    assert np.array_equal(nl.shift, g["shift"]) and np.array_equal(nl.rev, g["rev"])
    r = oracle.step(model, batch, nl, g["params"])
    np.testing.assert_allclose(r.E, g["E"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(r.F, g["F"], rtol=1e-10, atol=1e-12 * np.abs(g["F"]).max())
    assert abs(r.loss - g["loss"][0]) <= 1e-11 * abs(g["loss"][0])
    assert np.abs(r.grad - g["grad"]).max() <= 1e-11 * np.abs(g["grad"]).max()


@pytest.mark.parametrize("name", CASES)
def test_ledger_identity(oracle, name):
    """Eq. (2): dL/dtheta = BE merged first-order term + BF second-order term."""
    model, batch, g = load_case(oracle, name)
    r = oracle.step(model, batch, oracle.build_nbrlist(model, batch), g["params"])
    np.testing.assert_allclose(r.grad1 + r.grad2, r.grad, rtol=0, atol=1e-14 * np.abs(r.grad).max())
    assert np.abs(r.grad2).max() > 0 and np.abs(r.grad1).max() > 0


def test_forces_are_minus_energy_gradient(oracle):
    model, batch, g = load_case(oracle, "tiny")
    nl = oracle.build_nbrlist(model, batch)
    r = oracle.step(model, batch, nl, g["params"])
    eps = 1e-5
    for i in range(batch.n_atoms):
        for k in range(3):
            e = []
            for sgn in (+1, -1):
                p = batch.pos.copy()
                p[i, k] += sgn * eps
                b2 = oracle.Batch(p, batch.species, batch.struct_id, batch.cell, batch.E_target, batch.F_target)
                e.append(oracle.energy(model, b2, oracle.build_nbrlist(model, b2), g["params"]).sum())
            assert abs(-(e[0] - e[1]) / (2 * eps) - r.F[i, k]) < 1e-7 * max(1.0, abs(r.F).max())


def test_trace_is_consistent(oracle):
    """The per-unit boundary trace ends in the readout/embedding seeds."""
    model, batch, g = load_case(oracle, "two_struct")
    r = oracle.step(model, batch, oracle.build_nbrlist(model, batch), g["params"], want_trace=True)
    assert r.trace.shape == (model.n_units, 8, batch.n_atoms, model.H)
    assert np.abs(r.trace[1, 0]).max() > 0 and np.abs(r.trace[model.n_units - 2, 6]).max() > 0


@pytest.mark.parametrize("n,rho,seed", [(64, 0.095, 7), (256, 0.095, 701), (250, 0.095, 3), (4096, 0.19, 9)])
def test_oracle_synth_matches_product(janus, oracle, n, rho, seed):
    """The oracle's own synthetic-input restatement (used by bench.py's CPU
    reference arm, which must not load the product library) is bit-identical
    to the product's janus_synth_cell / janus_synth_params."""
    pos, sp, box, Et, Ft = oracle.synth_cell(n, rho, 4, seed)
    p2, s2, b2, E2, F2 = janus.synth_cell(n, rho, 4, seed)
    assert box == b2 and Et == E2
    assert np.array_equal(pos, p2) and np.array_equal(sp, s2) and np.array_equal(Ft, F2)
    for L, H in ((4, 64), (2, 256)):
        om = oracle.Model(L=L, H=H)
        jm = janus.Model(L=L, H=H)
        assert np.array_equal(oracle.synth_params(om, seed), jm.synth_params(seed))
