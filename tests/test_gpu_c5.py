"""configs[4] stress case at full size: 4096-atom periodic cells at rho 0.19
(~100 neighbours, ~410k directed edges per micro-batch), tf32 tensor-core
path, device-built neighbour lists, 8-stage WaveK on one GPU.  The CPU oracle
is too slow at this size, so parity uses size-independent properties:

* an 8-stage WaveK pipeline equals the single-stage step BIT FOR BIT
  (energies, forces, gradients, updated parameters);
* Newton's third law: per structure the forces sum to ~0 (every edge adds
  q_e u_e to F_i and its reverse subtracts it from F_j);
* translation invariance: a rigid shift of all atoms (positions re-wrapped
  into the box) leaves E within tf32 tolerance and F within 2e-2 of max |F|.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
N_ATOMS, RHO = 4096, 0.19


@pytest.fixture(scope="module")
def setup(janus, has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")
    m = janus.Model(L=4, H=64, R=64, precision=janus.PREC_TF32)
    params = m.synth_params(5)
    cells = [janus.synth_cell(N_ATOMS, RHO, m.n_species, 4000 + i) for i in range(2)]
    return m, params, cells


def batch(janus, cell, shift=None):
    pos, sp, L, Et, Ft = cell
    if shift is not None:
        pos = np.mod(pos + np.asarray(shift), L)
    return janus.Batch(pos, sp, np.zeros(len(pos), np.int32), [L], [Et], Ft, nl="device")


def run(janus, m, params, batches, P, method, k=1):
    t = janus.Trainer(m, params, P, method, len(batches), k=k, max_atoms=N_ATOMS, max_edges=N_ATOMS * 130,
                      max_struct=1, lanes=1)  # same lanes: same tiles and tiles per CTA
    t.load_many(batches)
    st = t.step(lr=1e-3)
    E = [t.stage(P - 1).energy(i, 1)[0][0] for i in range(len(batches))]
    F = [t.stage(0).forces(i, N_ATOMS)[0] for i in range(len(batches))]
    out = (st.loss, np.array(E), F, t.grads(), t.params())
    t.close()
    return out


def test_c5_pipeline_bit_identical_and_physics(janus, setup):
    m, params, cells = setup
    bs = [batch(janus, c) for c in cells]
    l1, E1, F1, g1, p1 = run(janus, m, params, bs, 1, janus.METHOD_SYMFOLD)
    l8, E8, F8, g8, p8 = run(janus, m, params, bs, 8, janus.METHOD_WAVEK, k=2)
    assert l1 == l8 and np.array_equal(E1, E8) and np.array_equal(g1, g8) and np.array_equal(p1, p8)
    assert all(np.array_equal(a, b) for a, b in zip(F1, F8))
    for F in F1:
        assert np.isfinite(F).all() and np.abs(F).max() > 0
        assert np.abs(F.sum(0)).max() < 1e-3 * np.abs(F).sum(0).max() + 1e-4
    # rigid translation (re-wrapped): same energy and forces within tf32 tolerance
    shifted = [batch(janus, c, shift=(1.37, -0.61, 2.9)) for c in cells]
    _, Es, Fs, _, _ = run(janus, m, params, shifted, 1, janus.METHOD_SYMFOLD)
    assert np.abs(Es - E1).max() <= 2e-3 * np.abs(E1).max()
    for a, b in zip(Fs, F1):
        assert np.abs(a - b).max() <= 2e-2 * np.abs(b).max()
