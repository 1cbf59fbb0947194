"""The schedule executor (C++ janus_trainer) on one GPU: P pipeline stages as
virtual devices with their own streams and a D2D transport.

* SymFold and WaveK at any P produce BIT-IDENTICAL gradients and updated
  parameters to P=1: per-micro-batch gradient ledgers are reduced in a fixed
  order, so neither P nor the schedule order changes a single rounding.
* 1F1B-2nd (recompute + replicated parameters + pairwise sum) matches the
  oracle within the fp32 tolerance.
* CUDA-graph replay equals eager issue bit-for-bit.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL_G = 1e-4


@pytest.fixture(scope="module")
def data(janus, oracle, has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")
    m = janus.Model(L=2, H=64, R=64)
    params = m.synth_params(21)
    batches = [janus.synth_batch(m, [n], 0.095, 100 + i) for i, n in enumerate([32, 40, 27, 36])]
    om = oracle.Model(L=m.L, H=m.H, R=m.R, n_species=m.n_species, r_c=m.r_c, w_E=m.w_E, w_F=m.w_F)
    g = np.zeros(m.param_count())
    loss = 0.0
    for b in batches:
        ob = oracle.Batch(b.pos, b.species, b.struct_id, b.cell, b.E_target.astype(float), b.F_target.astype(float))
        r = oracle.step(om, ob, oracle.build_nbrlist(om, ob), params.astype(float))
        g += r.grad
        loss += r.loss
    return m, params, batches, g, loss


def reduced_grad(janus, stage):
    ptr, n = ctypes.c_void_p(), ctypes.c_int64()
    fn = janus.lib().janus_stage_grad_buffer
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    janus.check(fn(stage.h, ctypes.byref(ptr), ctypes.byref(n)))
    out = np.zeros(n.value, np.float32)
    rt = janus.cudart()
    assert rt.cudaDeviceSynchronize() == 0
    assert rt.cudaMemcpy(out.ctypes.data, ptr.value, out.nbytes, 2) == 0
    return out


def run(janus, m, params, batches, P, method, k=1, graphs=False, timeline=False, steps=1):
    t = janus.Trainer(m, params, P, method, len(batches), k=k, max_atoms=64, max_edges=64 * 120,
                      graphs=graphs, timeline=timeline)
    for i, b in enumerate(batches):
        t.load(i, b)
    stats = [t.step(lr=1e-3) for _ in range(steps)]
    g = np.concatenate([reduced_grad(janus, t.stage(b)) for b in range(P)])
    p = t.params()
    return t, g, p, stats


def test_symfold_p1_matches_oracle(janus, data):
    m, params, batches, g_ref, loss_ref = data
    t, g, p, st = run(janus, m, params, batches, 1, janus.METHOD_SYMFOLD)
    assert np.abs(g - g_ref).max() / np.abs(g_ref).max() < TOL_G
    assert abs(st[0].loss - loss_ref) < 1e-5 * abs(loss_ref)
    assert st[0].makespan_ms > 0 and st[0].kernel_launches > 0
    t.close()


@pytest.mark.parametrize("P,method,k", [(2, 0, 1), (4, 0, 1), (4, 1, 2), (4, 1, 4), (6, 0, 1), (2, 4, 1), (4, 4, 1)])
def test_pipeline_bit_identical_to_p1(janus, data, P, method, k):
    m, params, batches, g_ref, _ = data
    t1, g1, p1, _ = run(janus, m, params, batches, 1, janus.METHOD_SYMFOLD)
    tp, gp, pp, st = run(janus, m, params, batches, P, method, k)
    assert np.array_equal(g1, gp) and np.array_equal(p1, pp)
    assert st[0].p2p_bytes > 0
    t1.close()
    tp.close()


@pytest.mark.parametrize("P", [2, 4])
def test_onef1b_2nd_matches_oracle(janus, data, P):
    m, params, batches, g_ref, loss_ref = data
    t, g, p, st = run(janus, m, params, batches, P, janus.METHOD_ONEF1B)
    assert np.abs(g - g_ref).max() / np.abs(g_ref).max() < TOL_G
    # the force replicas received the same summed gradient and took the same step
    for b in range(P):
        assert np.array_equal(t.stage(b).params(), t.stage(b, force_replica=True).params())
    t1, _, p1, _ = run(janus, m, params, batches, 1, janus.METHOD_SYMFOLD)
    assert np.abs(p - p1).max() < 1e-5
    t.close()
    t1.close()


def test_graph_replay_equals_eager(janus, data):
    m, params, batches, _, _ = data
    ta, ga, pa, _ = run(janus, m, params, batches, 4, janus.METHOD_WAVEK, k=2, steps=3)
    tb, gb, pb, _ = run(janus, m, params, batches, 4, janus.METHOD_WAVEK, k=2, graphs=True, steps=3)
    assert np.array_equal(ga, gb) and np.array_equal(pa, pb)
    ta.close()
    tb.close()


def test_timeline_and_bubble(janus, data):
    m, params, batches, _, _ = data
    P = 4
    t, _, _, st = run(janus, m, params, batches, P, janus.METHOD_SYMFOLD, timeline=True)
    tl = t.timeline()
    assert len(tl) == 4 * P * len(batches)  # one record per compute instruction
    assert (tl[:, 4] >= tl[:, 3]).all()
    s = st[0]
    assert 0.0 <= s.bubble_ratio < 1.0
    assert all(s.busy_ms[d] > 0 for d in range(P))
    t.close()


@pytest.mark.parametrize("P,lanes", [(1, 4), (4, 3)])
def test_lanes_bit_identical(janus, data, P, lanes):
    """Overlapping independent micro-batches on several streams of a device
    changes nothing: gradient ledgers are per micro-batch, reduced in order."""
    m, params, batches, _, _ = data
    t1, g1, p1, _ = run(janus, m, params, batches, P, janus.METHOD_SYMFOLD)
    t = janus.Trainer(m, params, P, janus.METHOD_SYMFOLD, len(batches), max_atoms=64, max_edges=64 * 120,
                      lanes=lanes, graphs=True)
    for i, b in enumerate(batches):
        t.load(i, b)
    t.step(lr=1e-3)
    g = np.concatenate([reduced_grad(janus, t.stage(b)) for b in range(P)])
    assert np.array_equal(g, g1) and np.array_equal(t.params(), p1)
    t.close()
    t1.close()


@pytest.mark.parametrize("graphs", [False, True])
def test_pipelined_loads_bit_identical(janus, data, graphs):
    """Input pipelining (loads of step k+1 queued behind step k via
    step_async/wait, as bench.py's e2e loop does) changes nothing: every step
    sees its own freshly uploaded batches; losses and parameters match the
    synchronous load+step loop bit for bit.  Step k+1 uses different batches
    (reversed order) so a stale geometry or tile table would show."""
    m, params, batches, _, _ = data
    order = [batches, batches[::-1], batches]

    def make():
        return janus.Trainer(m, params, 2, janus.METHOD_SYMFOLD, len(batches), k=1, max_atoms=64,
                             max_edges=64 * 120, graphs=graphs, lanes=2)

    ta = make()
    la = []
    for bs in order:
        for i, b in enumerate(bs):
            ta.load(i, b)
        la.append(ta.step().loss)
    pa = ta.params()

    tb = make()
    lb = []
    for i, b in enumerate(order[0]):
        tb.load(i, b)
    tb.step_async()
    for bs in order[1:]:
        for i, b in enumerate(bs):
            tb.load(i, b)
        lb.append(tb.wait().loss)
        tb.step_async()
    lb.append(tb.wait().loss)
    pb = tb.params()
    assert la == lb
    assert np.array_equal(pa, pb)
    with pytest.raises(janus.JanusError):
        tb.wait()  # nothing in flight
    ta.close()
    tb.close()


@pytest.mark.parametrize("P,method,k,atoms", [(4, 1, 8, 64), (2, 0, 1, 64), (4, 1, 8, 128), (3, 0, 1, 128)])
def test_tensor_core_pipeline_lanes_bit_identical(janus, P, method, k, atoms):
    """The N>1 bench configuration on one GPU: tensor-core kernels, device-built
    neighbour lists, P pipeline stages with 8 compute lanes per stage and
    double-buffered loads — bit-identical to one stage with the same lanes.
    128-atom cells take the tcgen05 upd kernels (upd_tc.cuh), including the
    unfused next-v products at stage starts; 64-atom cells the SIMT ones."""
    if not janus.device_count():
        pytest.skip("no GPU")
    m = janus.Model(L=2, H=64, R=64, precision=janus.PREC_TF32)
    params = m.synth_params(8)
    bs = [janus.synth_batch(m, [atoms + 8 * (i % 3)], 0.095, 300 + i, device_nl=True) for i in range(16)]
    out = []
    for PP, meth, kk in ((1, janus.METHOD_SYMFOLD, 1), (P, method, k)):
        t = janus.Trainer(m, params, PP, meth, len(bs), k=kk, max_atoms=atoms + 32, max_edges=(atoms + 32) * 80, lanes=8,
                          graphs=True)
        t.load_many(bs)
        losses = []
        for _ in range(2):
            t.step_async(lr=1e-3)
            t.load_many(bs)  # next step's loads beside the step in flight
            losses.append(t.wait().loss)
        out.append((losses, t.params(), t.grads()))
        t.close()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])


@pytest.mark.parametrize("P,method", [(1, 0), (2, 1)])
def test_tensor_core_trainer_ragged_matches_oracle(janus, data, P, method):
    """Tensor-core mode through the executor on ragged micro-batches (27..40
    atoms: every micro-batch has its own pair count, pair-kernel grid and
    partial count): the summed gradient matches the fp64 oracle within the
    tensor-core tolerance (tests/test_gpu_tf32.py: 2e-2 of the max)."""
    m, params, batches, g_ref, _ = data
    m_tc = janus.Model(L=m.L, H=m.H, R=m.R, precision=janus.PREC_TF32)
    t, g, _, _ = run(janus, m_tc, params, batches, P, method, k=2 if method == 1 else 1)
    t.close()
    err = float(np.abs(g - g_ref).max() / np.abs(g_ref).max())
    assert err < 2e-2, err


@pytest.mark.parametrize("graphs", [False, True])
def test_two_steps_in_flight_bit_identical(janus, data, graphs):
    """bench.py's e2e loop keeps two steps in flight (step k+1 issued before
    step k's loss is read; step k+2's loads issued while k+1 runs): losses
    (each read from its own step's snapshot) and parameters match the
    synchronous loop bit for bit, with the batches changing every step."""
    m, params, batches, _, _ = data
    order = [batches, batches[::-1], batches, batches[::-1], batches]

    def make():
        return janus.Trainer(m, params, 1, janus.METHOD_SYMFOLD, len(batches), k=1, max_atoms=64,
                             max_edges=64 * 120, graphs=graphs, lanes=2)

    ta = make()
    la = []
    for bs in order:
        ta.load_many(bs)
        la.append(ta.step().loss)
    pa = ta.params()

    tb = make()
    lb = []
    tb.load_many(order[0])
    tb.step_async()
    tb.load_many(order[1])
    tb.step_async()
    with pytest.raises(janus.JanusError):
        tb.step_async()  # at most two in flight
    for bs in order[2:]:
        lb.append(tb.wait().loss)
        tb.load_many(bs)
        tb.step_async()
    lb.append(tb.wait().loss)
    lb.append(tb.wait().loss)
    pb = tb.params()
    assert la == lb
    assert np.array_equal(pa, pb)
    ta.close()
    tb.close()


@pytest.mark.parametrize("P,method,k", [(2, 0, 1), (4, 0, 1), (4, 1, 4), (4, 2, 1), (4, 4, 1)])
def test_slot_pool_folds_memory_bit_identically(janus, data, P, method, k):
    """The activation arena is a pool sized by the schedule's live
    micro-batches (include/janus/slots.hpp): fewer slots and
    bytes than one slot per micro-batch, the predicted slot count per device,
    and the same bits (reused slots wait for their previous occupant)."""
    m, params, batches, _, _ = data
    batches8 = batches + batches
    res = {}
    for unfolded in (False, True):
        t = janus.Trainer(m, params, P, method, len(batches8), k=k, max_atoms=64, max_edges=64 * 120,
                          unfolded=unfolded)
        for i, b in enumerate(batches8):
            t.load(i, b)
        st = [t.step(lr=1e-3) for _ in range(2)]
        g = np.concatenate([reduced_grad(janus, t.stage(b)) for b in range(P)])
        res[unfolded] = (g, t.params(), st[-1], t.schedule_text())
        t.close()
    g0, p0, s0, text = res[False]
    g1, p1, s1, _ = res[True]
    assert np.array_equal(g0, g1) and np.array_equal(p0, p1)
    pred = janus.slot_pool(text, onef1b=(method == janus.METHOD_ONEF1B), local=True)
    assert list(s0.act_slots[:P]) == pred
    assert all(s1.act_slots[d] == len(batches8) for d in range(P))
    assert sum(s0.act_bytes[:P]) <= sum(s1.act_bytes[:P])
    if sum(pred) < P * len(batches8):  # WaveK(k=P) keeps 2P = all 8 micro-batches live
        assert sum(s0.act_bytes[:P]) < sum(s1.act_bytes[:P])
        assert max(s0.peak_bytes[:P]) < max(s1.peak_bytes[:P])
