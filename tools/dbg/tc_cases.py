import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2605_18404_b200 as janus
def run(prec, b):
    m = janus.Model(L=2, H=64, R=64, precision=prec)
    params = m.synth_params(11)
    st = janus.Stage(m, params, 0, m.n_units, max_atoms=256, max_edges=256 * 120, max_struct=4)
    st.load(0, b)
    st.fe(0)
    E, _ = st.energy(0, b.n_struct)
    st.ff(0)
    F, _ = st.forces(0, b.n_atoms)
    st.close()
    return E, F
m0 = janus.Model(L=2)
for name, sizes, rho in [("dense200", [200], 0.19), ("sparse200", [200], 0.095), ("dense64", [64], 0.19), ("dense100", [100], 0.19), ("sparse256", [256], 0.095)]:
    b = janus.synth_batch(m0, sizes, rho, 4)
    deg = np.diff(b.row_ptr)
    E0, F0 = run(janus.PREC_FP32, b)
    E1, F1 = run(janus.PREC_TF32, b)
    print(name, "deg max", deg.max(), "mean", deg.mean(), "E rel", float(np.abs(E1 - E0).max() / np.abs(E0).max()), "F rel", float(np.abs(F1 - F0).max() / np.abs(F0).max()), flush=True)
