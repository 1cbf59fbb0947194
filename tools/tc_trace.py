"""Phase trace of the tensor-core edge kernels (profiling aid).

  make TRACE=1 lib && JANUS_LIB=build/trace/libjanus_b200.so python tools/tc_trace.py

Runs one 256-atom micro-batch through the four phases; the traced build
prints clock64 deltas between the TC_MARK points of edge_tc.cuh."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_18404_b200 as janus  # noqa: E402

m = janus.Model(L=2, H=64, R=64, precision=janus.PREC_TF32)
params = m.synth_params(11)
b = janus.synth_batch(m, [256], 0.095, 9)
st = janus.Stage(m, params, 0, m.n_units, max_atoms=256, max_edges=256 * 120, max_struct=1)
st.load(0, b)
for rep in range(3):
    for ph in ("fe", "ff", "bf", "be"):
        getattr(st, ph)(0)
    janus.cudart().cudaDeviceSynchronize()
    print(f"--- rep {rep} done", flush=True)
st.close()
