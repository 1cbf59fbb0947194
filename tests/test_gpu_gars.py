"""GARS regroups structures without changing the step gradient
(PAPER.md:743-744): a global batch of mixed-size cells packed by
pack-and-shuffle and by the greedy baseline trains (fp32 SIMT path, device
LM) to the same gradient as the fp64 oracle's per-structure sum."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gars_packing_preserves_gradient(janus, oracle, has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")
    m = janus.Model(L=2, H=64, R=64)
    params = m.synth_params(3)
    sizes = [27, 64, 32, 40, 27, 54, 36, 64, 30, 48, 27, 60]
    cells = [janus.synth_cell(n, 0.095, m.n_species, 900 + i) for i, n in enumerate(sizes)]
    om = oracle.Model(L=m.L, H=m.H, R=m.R, n_species=m.n_species, r_c=m.r_c, w_E=m.w_E, w_F=m.w_F)
    g_ref = np.zeros(m.param_count())
    for pos, sp, L, Et, Ft in cells:
        ob = oracle.Batch(pos, sp, np.zeros(len(pos), np.int32), [L], [Et], Ft.astype(float))
        g_ref += oracle.step(om, ob, oracle.build_nbrlist(om, ob), params.astype(float)).grad
    grads = []
    for greedy in (False, True):
        groups = [g for g, _ in janus.gars_pack(sizes, 4, 1, seed=5, greedy=greedy)]
        batches = []
        for g in groups:
            P = [cells[i][0] for i in g]
            batches.append(janus.Batch(np.concatenate(P), np.concatenate([cells[i][1] for i in g]),
                                       np.concatenate([np.full(len(cells[i][0]), s, np.int32) for s, i in enumerate(g)]),
                                       np.array([cells[i][2] for i in g]), np.array([cells[i][3] for i in g]),
                                       np.concatenate([cells[i][4] for i in g]), nl="device"))
        t = janus.Trainer(m, params, 2, janus.METHOD_SYMFOLD, 4, max_atoms=256, max_edges=256 * 80, max_struct=8)
        t.load_many(batches)
        t.step(lr=0.0)
        grads.append(t.grads())
        t.close()
    for g in grads:
        assert np.abs(g - g_ref).max() / np.abs(g_ref).max() < 1e-4
