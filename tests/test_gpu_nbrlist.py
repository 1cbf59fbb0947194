"""Device neighbour list (nbrlist.cu): the cell-list
build on the GPU is BIT-IDENTICAL to the host build (janus_nbrlist_build) and
to the oracle's (oracle/mlip_oracle.c mo_build_nbrlist) — row_ptr, col,
shift and rev — on the configs' cells, on boxes smaller than r_c (several
images), on multi-structure batches, on unwrapped positions and on dilute
cells with empty rows; a capacity overflow is a domain error.  A trainer whose
loads build the CSR on the device takes the same step, bit for bit, as one fed
the host CSR."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu(janus, has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")
    return janus


def cells(janus, sizes, rho, seed, r_c=5.0):
    P, SID, C = [], [], []
    for s, n in enumerate(sizes):
        pos, sp, L, Et, Ft = janus.synth_cell(n, rho, 4, seed * 1000003 + s)
        P.append(pos)
        SID.append(np.full(n, s, np.int32))
        C.append(L)
    return np.concatenate(P), np.concatenate(SID), np.array(C)


def assert_same(a, b):
    for x, y, name in zip(a, b, ("row_ptr", "col", "shift", "rev")):
        assert np.array_equal(np.asarray(x).ravel(), np.asarray(y).ravel()), name


CASES = [
    ("C1 64-atom cell (one cell, 27 images)", [64], 0.095),
    ("C2 256-atom fcc cell", [256], 0.095),
    ("C3 512-atom cell", [512], 0.095),
    ("C5 4096-atom dense cell", [4096], 0.19),
    ("C4 mixed sizes", [128, 250, 256, 432, 500, 1024], 0.095),
    ("box smaller than r_c (5x5x5 images)", [3, 5], 0.095),
    ("dilute, empty rows", [20], 0.004),
    # ~160 neighbours per atom: rows above nbrlist.cu's kPadCap (128) take the re-walk path
    ("very dense rows (> kPadCap)", [400], 0.30),
    ("dense rows over kSortCap (512)", [1200], 0.99),
]


@pytest.mark.parametrize("name,sizes,rho", CASES, ids=[c[0] for c in CASES])
def test_device_nbrlist_bit_exact(gpu, oracle, name, sizes, rho):
    janus = gpu
    pos, sid, cell = cells(janus, sizes, rho, 11)
    host = janus.nbrlist(pos, sid, cell, 5.0, max_edges=len(pos) * 700)
    dev = janus.nbrlist_device(pos, sid, cell, 5.0, max_edges=len(pos) * 700)
    assert_same(dev, host)
    if len(pos) <= 1100:  # the oracle's O(N^2) build: keep the CPU part short
        om = oracle.Model(L=1, H=64, R=64, n_species=4, r_c=5.0, w_E=1.0, w_F=10.0)
        ob = oracle.Batch(pos, np.zeros(len(pos), np.int32), sid, cell, np.zeros(len(cell)),
                          np.zeros((len(pos), 3)))
        o = oracle.build_nbrlist(om, ob)
        assert_same(dev, (o.row_ptr, o.col, o.shift, o.rev))
    if "empty" in name:
        assert (np.diff(dev[0]) == 0).any()


def test_device_nbrlist_unwrapped_positions(gpu):
    """Positions outside [0, L): the image filter |s| <= ceil(r_c/L) of the
    host build is kept, so the CSR still matches bit for bit."""
    janus = gpu
    pos, sid, cell = cells(janus, [256, 64], 0.095, 5)
    rng = np.random.default_rng(3)
    for a in range(len(pos)):
        pos[a] += rng.integers(-2, 3, size=3) * cell[sid[a]]
    assert_same(janus.nbrlist_device(pos, sid, cell, 5.0), janus.nbrlist(pos, sid, cell, 5.0))


def test_device_nbrlist_capacity_error(gpu):
    janus = gpu
    pos, sid, cell = cells(janus, [256], 0.095, 2)
    with pytest.raises(janus.JanusError) as e:
        janus.nbrlist_device(pos, sid, cell, 5.0, max_edges=1000)
    assert e.value.code == 1 and "max_edges" in str(e.value)


@pytest.mark.parametrize("graphs,many", [(False, False), (True, False), (True, True)])
def test_trainer_device_lm_bit_identical(gpu, graphs, many):
    """Loads without a CSR (device LM, side stream, pipelined behind a step)
    give the same losses, gradients and parameters as host-CSR loads."""
    janus = gpu
    m = janus.Model(L=2, H=64, R=64, precision=janus.PREC_TF32)
    params = m.synth_params(4)
    sizes = [64, 108, 128, 64]
    host = [janus.synth_batch(m, [n], 0.095, 40 + i) for i, n in enumerate(sizes)]
    dev = [janus.synth_batch(m, [n], 0.095, 40 + i, device_nl=True) for i, n in enumerate(sizes)]
    out = []
    for batches in (host, dev):
        t = janus.Trainer(m, params, 1, janus.METHOD_SYMFOLD, len(batches), max_atoms=128, max_edges=128 * 120,
                          graphs=graphs, lanes=2)
        losses = []

        def load_all():
            if many:  # one batched device build for all micro-batches
                t.load_many(batches)
            else:
                for i, b in enumerate(batches):
                    t.load(i, b)
        load_all()
        for step in range(3):
            t.step_async(lr=1e-3)
            if step < 2:  # next step's loads queued behind the step in flight
                load_all()
            losses.append(t.wait().loss)
        out.append((losses, t.params(), t.grads()))
        t.close()
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])
