"""Generic-width stage path (csrc/stage_wide.inc + wide.cuh): configs[2]'s
deep model (H=256) and any H in {64, 128, 256}, against the fp64 oracle.

* fp32 (PREC_FP32, plain fp32 GEMMs): the north-star tolerances — E relative
  1e-5, F and gradients 1e-4 of the max magnitude.
* tf32 (PREC_TF32: the same GEMMs on tf32 tensor-core math, fp32 accumulate):
  E 2e-3, F and gradients 2e-2 (the tensor-core tolerance of
  tests/test_gpu_tf32.py).
* fp32-emulated (PREC_FP32_EMU: BF16x9 fp32 emulation on the tensor cores):
  the fp32 tolerances.
* Staged (P virtual stages, mid-layer splits) == unstaged, bit for bit, and
  pooled activation slots == one slot per micro-batch.
* At H=64 the generic path agrees with the fused H=64 kernels.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


def oracle_refs(janus, oracle, m, params, batches):
    om = oracle.Model(L=m.L, H=m.H, R=m.R, n_species=m.n_species, r_c=m.r_c, w_E=m.w_E, w_F=m.w_F)
    refs = []
    for b in batches:
        ob = oracle.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target.astype(np.float64),
                          b.F_target.astype(np.float64))
        nl = oracle.build_nbrlist(om, ob)
        refs.append(oracle.step(om, ob, nl, params.astype(np.float64)))
    return refs


def run_stage(janus, m, params, batches, max_atoms=64):
    st = janus.Stage(m, params, 0, m.n_units, max_atoms=max_atoms, max_edges=max_atoms * 200, max_struct=4,
                     n_mb=len(batches), n_slots=len(batches))
    for i, b in enumerate(batches):
        st.load(i, b)
    for ph in ("fe", "ff", "bf", "be"):
        for i in range(len(batches)):
            getattr(st, ph)(i)
    return st


@pytest.mark.parametrize("H,R,prec", [(64, 64, 0), (128, 32, 0), (256, 64, 0), (256, 64, 1), (128, 64, 1), (64, 64, 1),
                                      (64, 64, 2), (256, 64, 2)])
def test_wide_matches_oracle(janus, oracle, has_gpu, H, R, prec):
    if not has_gpu:
        pytest.skip("no GPU")
    tol_e, tol_f = (2e-3, 2e-2) if prec == janus.PREC_TF32 else (1e-5, 1e-4)
    m = janus.Model(L=2, H=H, R=R, precision=prec, generic=True)
    params = m.synth_params(5)
    batches = [janus.synth_batch(m, [24, 30], 0.095, 31), janus.synth_batch(m, [40], 0.095, 32)]
    try:
        st = run_stage(janus, m, params, batches)
    except janus.JanusError as ex:  # BF16x9 emulation: the process's libcublas may predate 12.9
        if "needs cuBLAS >= 12.9" in str(ex):
            pytest.skip(str(ex))
        raise
    refs = oracle_refs(janus, oracle, m, params, batches)
    for i, (b, r) in enumerate(zip(batches, refs)):
        E, lE = st.energy(i, b.n_struct)
        F, lF = st.forces(i, b.n_atoms)
        assert rel(E, r.E) < tol_e, (H, rel(E, r.E))
        assert rel(F, r.F) < tol_f, (H, rel(F, r.F))
        g1, g2 = st.grads(1, i), st.grads(2, i)
        assert rel(g1, r.grad1) < tol_f, (H, rel(g1, r.grad1))
        assert rel(g2, r.grad2) < tol_f, (H, rel(g2, r.grad2))
        for u in range(m.n_units):  # localise: every unit's block
            o0, o1 = m.unit_offset(u), m.unit_offset(u + 1)
            g = g1[o0:o1] + g2[o0:o1]
            scale = max(np.abs(r.grad).max(), 1e-30)
            assert np.abs(g - r.grad[o0:o1]).max() / scale < tol_f, f"H={H} unit {u}"
    st.close()


def test_wide_h64_agrees_with_fused_kernels(janus, has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")
    out = {}
    for generic in (False, True):
        m = janus.Model(L=2, H=64, R=64, generic=generic)
        params = m.synth_params(9)
        batches = [janus.synth_batch(m, [36], 0.095, 41)]
        st = run_stage(janus, m, params, batches)
        out[generic] = (st.energy(0, 1)[0], st.forces(0, 36)[0], st.grads(0, 0))
        st.close()
    for a, b, tol in zip(out[False], out[True], (1e-5, 1e-4, 1e-4)):
        assert rel(a, b) < tol


@pytest.mark.parametrize("P,method,prec", [(2, 0, 0), (4, 0, 0), (4, 1, 0), (3, 4, 0), (3, 0, 1), (4, 1, 1)])
def test_wide_pipeline_bit_identical(janus, has_gpu, P, method, prec):
    """L=3, H=256: staged (incl. mid-layer splits), pooled slots, WaveK /
    Hanayo orders — all equal to P=1 bit for bit (prec 1: the TMA-fed
    tcgen05 GEMMs of gemm_tc.cuh)."""
    if not has_gpu:
        pytest.skip("no GPU")
    m = janus.Model(L=3, H=256, R=64, generic=True, precision=prec)
    params = m.synth_params(13)
    batches = [janus.synth_batch(m, [n], 0.095, 50 + i) for i, n in enumerate([32, 40, 27, 36, 30, 33])]
    res = []
    for PP, meth in ((1, 0), (P, method)):
        t = janus.Trainer(m, params, PP, meth, len(batches), k=2, max_atoms=64, max_edges=64 * 120)
        for i, b in enumerate(batches):
            t.load(i, b)
        s = [t.step(lr=1e-3) for _ in range(2)]
        res.append((t.params(), s[-1].loss))
        t.close()
    assert np.array_equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1]
