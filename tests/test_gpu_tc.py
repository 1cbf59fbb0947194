"""tcgen05 layer self-test on the B200: the descriptor encodings in
csrc/tc.cuh (no-swizzle core-matrix tiles, K-major and MN-major views,
kind::tf32) against numpy, and the TMEM row->lane map of M=64 accumulators."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def probe(janus, M, N, K, a_mn, b_mn, A, B, swap=0, layout=0):
    fn = janus.lib().janus_tc_probe
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    args = np.array([M, N, K, a_mn, b_mn, A.shape[0], A.shape[1], B.shape[0], B.shape[1], swap, layout], np.int32)
    D = np.zeros((128, N), np.float32)
    janus.check(fn(args.ctypes.data, A.ctypes.data, B.ctypes.data, D.ctypes.data))
    return D


def tf32(x):
    b = np.ascontiguousarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32).astype(np.float64)


def lane_map(D, G):
    lanes, errs = [], []
    for r in range(G.shape[0]):
        e = np.abs(D - G[r][None, :]).max(axis=1)
        lanes.append(int(e.argmin()))
        errs.append(float(e.min()))
    return lanes, max(errs) / np.abs(G).max()


CASES = {
    # name: (M, N, K, a_mn, b_mn, A shape, B shape, reference(A, B) -> G[M][N])
    "kmajor_m128": (128, 64, 64, 0, 0, (128, 64), (64, 64), lambda A, B: A @ B.T),
    "kmajor_m64": (64, 64, 128, 0, 0, (64, 128), (64, 128), lambda A, B: A @ B.T),
    "amn_m128": (128, 64, 64, 1, 0, (64, 128), (64, 64), lambda A, B: A.T @ B.T),
    "bmn_m128": (128, 64, 64, 0, 1, (128, 64), (64, 64), lambda A, B: A @ B),
    "mn_m64": (64, 64, 128, 1, 1, (128, 64), (128, 64), lambda A, B: A.T @ B),
}


MN = {"amn_m128", "bmn_m128", "mn_m64"}  # tcgen05 transpose bit with kind::tf32: measured to return zeros


@pytest.mark.parametrize("name", [n for n in CASES if n not in MN])
def test_probe(janus, has_gpu, name):
    if not has_gpu:
        pytest.skip("no GPU")
    M, N, K, amn, bmn, sa, sb, ref = CASES[name]
    rng = np.random.default_rng(hash(name) % 1000)
    A = rng.normal(size=sa).astype(np.float32)
    B = rng.normal(size=sb).astype(np.float32)
    D = probe(janus, M, N, K, amn, bmn, A, B)
    G = ref(tf32(A), tf32(B))
    lanes, err = lane_map(D, G)
    print(f"{name}: rel err {err:.2e}; row->lane {lanes}")
    assert err < 1e-3
    if M == 128:
        assert lanes == list(range(128))


@pytest.mark.parametrize("name", ["amn_m128", "bmn_m128", "mn_m64"])
def test_probe_mn_swapped(janus, has_gpu, name):
    """Diagnostic: MN-major with LBO/SBO exchanged."""
    if not has_gpu:
        pytest.skip("no GPU")
    M, N, K, amn, bmn, sa, sb, ref = CASES[name]
    rng = np.random.default_rng(7)
    A = rng.normal(size=sa).astype(np.float32)
    B = rng.normal(size=sb).astype(np.float32)
    D = probe(janus, M, N, K, amn, bmn, A, B, swap=1)
    lanes, err = lane_map(D, ref(tf32(A), tf32(B)))
    print(f"{name} swapped: rel err {err:.2e}; |D| max {np.abs(D).max():.3f}")
    # documents the finding that drives edge_tc.cuh's transposed tiles
    assert np.abs(D).max() == 0.0


@pytest.mark.parametrize("name", [n for n in CASES if n not in MN])
def test_probe_sw128(janus, has_gpu, name):
    """SWIZZLE_128B tiles: K-major and MN-major views of [row][col] slabs."""
    if not has_gpu:
        pytest.skip("no GPU")
    M, N, K, amn, bmn, sa, sb, ref = CASES[name]
    rng = np.random.default_rng(11)
    A = rng.normal(size=sa).astype(np.float32)
    B = rng.normal(size=sb).astype(np.float32)
    D = probe(janus, M, N, K, amn, bmn, A, B, layout=2)
    lanes, err = lane_map(D, ref(tf32(A), tf32(B)))
    print(f"{name} sw128: rel err {err:.2e}; |D| max {np.abs(D).max():.3f}; lanes[:20] {lanes[:20]}")
    assert err < 1e-3


def gemm_probe(janus, rows, K, N, pair, A, W):
    fn = janus.lib().janus_gemm_tc_probe
    fn.argtypes = [ctypes.c_int32] * 4 + [ctypes.c_void_p] * 3
    A = np.ascontiguousarray(A, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    D = np.zeros((A.shape[0], N), np.float32)
    janus.check(fn(rows, K, N, pair, A.ctypes.data, W.ctypes.data, D.ctypes.data))
    return D


@pytest.mark.parametrize("rows,K,N,pair", [(200, 64, 256, 0), (300, 256, 256, 0), (128, 256, 64, 0), (77, 64, 128, 0),
                                           (100, 64, 256, 1), (130, 256, 256, 1), (64, 32, 64, 1)])
def test_tma_gemm_matches_numpy(janus, has_gpu, rows, K, N, pair):
    """gemm_tc.cuh: TMA (SWIZZLE_128B tensor maps) + tcgen05 kind::tf32,
    warp-specialised pipeline; pair mode stacks [value; derivative] rows.
    Against numpy on tf32-truncated inputs (fp32 accumulate)."""
    if not has_gpu:
        pytest.skip("no GPU")
    rng = np.random.default_rng(rows * 7 + K)
    A = rng.standard_normal(((2 if pair else 1) * rows, K)).astype(np.float32)
    W = rng.standard_normal((N, K)).astype(np.float32)
    D = gemm_probe(janus, rows, K, N, pair, A, W)
    ref = tf32(A) @ tf32(W).T
    assert np.abs(D - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("rows,K,N,pair", [(200, 64, 256, 0), (300, 256, 256, 0), (77, 64, 128, 0), (100, 64, 256, 1),
                                           (130, 256, 64, 1)])
def test_tma_gemm_split3_is_fp32_accurate(janus, has_gpu, rows, K, N, pair):
    """gemm_tc.cuh 3xTF32 mode (Problem::split3, the fp32-tolerance path's
    per-pair products): against an fp64 reference it is ~fp32-accurate
    (4e-6 of max at K <= 256, the error scale of an fp32 accumulation), where
    single-pass tf32 is ~7e-4."""
    if not has_gpu:
        pytest.skip("no GPU")
    rng = np.random.default_rng(rows * 11 + K)
    A = rng.standard_normal(((2 if pair else 1) * rows, K)).astype(np.float32)
    W = rng.standard_normal((N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ W.astype(np.float64).T
    scale = np.abs(ref).max()
    D3 = gemm_probe(janus, rows, K, N, pair | 2, A, W)
    D1 = gemm_probe(janus, rows, K, N, pair, A, W)
    e3, e1 = np.abs(D3 - ref).max() / scale, np.abs(D1 - ref).max() / scale
    print(f"3xTF32 rel err {e3:.2e}, tf32 {e1:.2e}")
    assert e3 <= 4e-6
    assert e1 > 50 * e3
