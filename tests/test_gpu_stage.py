"""GPU parity of the four-phase step through the C ABI against the fp64 oracle.

Tolerances (fp32 SIMT parity mode, stated per BASELINE north star):
  E: relative 1e-5;  F and parameter gradients: 1e-4 of the max magnitude.
Staged execution (P stages on one GPU, ports moved by cudaMemcpy = the fake
transport of SURVEY.md §4) must equal P=1 bit-for-bit: every unit runs the
same kernels and the force/gradient accumulation orders do not depend on P.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_E, TOL_F, TOL_G = 1e-5, 1e-4, 1e-4


@pytest.fixture(scope="module")
def setup(janus, oracle, has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")
    m = janus.Model(L=2, H=64, R=64)
    params = m.synth_params(11)
    batches = [janus.synth_batch(m, [24, 30], 0.095, 3), janus.synth_batch(m, [40], 0.095, 4)]
    om = oracle.Model(L=m.L, H=m.H, R=m.R, n_species=m.n_species, r_c=m.r_c, w_E=m.w_E, w_F=m.w_F)
    refs = []
    for b in batches:
        ob = oracle.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target.astype(np.float64),
                          b.F_target.astype(np.float64))
        nl = oracle.build_nbrlist(om, ob)
        assert np.array_equal(nl.col, b.col)
        refs.append(oracle.step(om, ob, nl, params.astype(np.float64)))
    return m, params, batches, refs


def run_single(janus, m, params, batches, order=None):
    U = m.n_units
    st = janus.Stage(m, params, 0, U, max_atoms=64, max_edges=64 * 200, max_struct=4, n_mb=len(batches),
                     n_slots=len(batches))
    for i, b in enumerate(batches):
        st.load(i, b)
    # SymFold P=1 order for two micro-batches: FE0 FE1 FF0 BF0 FF1 BE0 BF1 BE1
    order = order or [("fe", 0), ("fe", 1), ("ff", 0), ("bf", 0), ("ff", 1), ("be", 0), ("bf", 1), ("be", 1)]
    for ph, mb in order:
        if mb < len(batches):
            getattr(st, ph)(mb)
    return st


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


def test_single_stage_matches_oracle(janus, setup):
    m, params, batches, refs = setup
    st = run_single(janus, m, params, batches)
    for i, (b, r) in enumerate(zip(batches, refs)):
        E, lE = st.energy(i, b.n_struct)
        F, lF = st.forces(i, b.n_atoms)
        assert rel(E, r.E) < TOL_E, (E, r.E)
        assert rel(F, r.F) < TOL_F
        assert abs(lE + lF - r.loss) < TOL_E * abs(r.loss) + 1e-4
        g1, g2, g = st.grads(1, i), st.grads(2, i), st.grads(0, i)
        assert rel(g1, r.grad1) < TOL_G, rel(g1, r.grad1)
        assert rel(g2, r.grad2) < TOL_G, rel(g2, r.grad2)
        assert rel(g, r.grad) < TOL_G
    gsum = st.grads(0, -1)
    assert rel(gsum, refs[0].grad + refs[1].grad) < TOL_G
    st.close()


def test_per_unit_gradients(janus, setup):
    """Localise errors: every unit's parameter block within tolerance."""
    m, params, batches, refs = setup
    st = run_single(janus, m, params, batches[:1], order=[("fe", 0), ("ff", 0), ("bf", 0), ("be", 0)])
    g = st.grads(0, 0)
    for u in range(m.n_units):
        o0, o1 = m.unit_offset(u), m.unit_offset(u + 1)
        scale = max(np.abs(refs[0].grad).max(), 1e-30)
        assert np.abs(g[o0:o1] - refs[0].grad[o0:o1]).max() / scale < TOL_G, f"unit {u}"
    st.close()


@pytest.mark.parametrize("cuts", [[0, 3, 6], [0, 2, 4, 6], [0, 1, 2, 3, 4, 5, 6], [0, 5, 6]])
def test_staged_equals_unstaged_bitwise(janus, setup, cuts):
    """P stages on one GPU (fake transport) == P=1, bit for bit.  Cuts at odd
    unit indices split a layer between msg and upd (payload carries m)."""
    m, params, batches, refs = setup
    b = batches[0]
    ref = run_single(janus, m, params, [b], order=[("fe", 0), ("ff", 0), ("bf", 0), ("be", 0)])
    stages = [janus.Stage(m, params, cuts[p], cuts[p + 1], max_atoms=64, max_edges=64 * 200, max_struct=4)
              for p in range(len(cuts) - 1)]
    P = len(stages)
    for s in stages:
        s.load(0, b)

    def move(src, sport, dst, dport):
        a, na = src.port(0, 0, sport)
        d, nd = dst.port(0, 0, dport)
        assert na == nd and na > 0
        janus.d2d(d, a, na)

    for p in range(P):
        stages[p].fe(0)
        if p + 1 < P:
            move(stages[p], janus.PORT_ACT_OUT, stages[p + 1], janus.PORT_ACT_IN)
    for p in reversed(range(P)):
        stages[p].ff(0)
        if p > 0:
            move(stages[p], janus.PORT_ADJ_OUT, stages[p - 1], janus.PORT_ADJ_IN)
    for p in range(P):
        stages[p].bf(0)
        if p + 1 < P:
            move(stages[p], janus.PORT_TAN_OUT, stages[p + 1], janus.PORT_TAN_IN)
    for p in reversed(range(P)):
        stages[p].be(0)
        if p > 0:
            move(stages[p], janus.PORT_BADJ_OUT, stages[p - 1], janus.PORT_BADJ_IN)
    E, _ = stages[-1].energy(0, b.n_struct)
    F, _ = stages[0].forces(0, b.n_atoms)
    E1, _ = ref.energy(0, b.n_struct)
    F1, _ = ref.forces(0, b.n_atoms)
    assert np.array_equal(E, E1) and np.array_equal(F, F1)
    g = np.concatenate([s.grads(0, 0) for s in stages])
    assert np.array_equal(g, ref.grads(0, 0))
    for s in stages:
        s.close()
    ref.close()


def test_adam_step(janus, oracle, setup):
    m, params, batches, refs = setup
    st = run_single(janus, m, params, batches)
    g = st.grads(0, -1).astype(np.float64)
    st.reduce_grads()
    st.optimizer_step(lr=1e-3)
    got = st.params()
    p = params.astype(np.float64).copy()
    m1, m2 = np.zeros_like(p), np.zeros_like(p)
    oracle.adam(p, m1, m2, g, 1e-3, 0.9, 0.999, 1e-8, 1)
    assert np.abs(got - p).max() < 1e-6
    st.close()
