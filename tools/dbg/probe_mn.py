"""tcgen05 MN-major operands: kind::tf32 (SWIZZLE_128B) vs kind::f16 bf16 (SWIZZLE_128B)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import paper_2605_18404_b200 as J
from test_gpu_tc import CASES, probe, tf32, lane_map
def bf16(x):
    b = np.ascontiguousarray(x, np.float32).view(np.uint32)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return b.view(np.float32).astype(np.float64)
for name in ("kmajor_m128", "kmajor_m64", "amn_m128", "bmn_m128", "mn_m64"):
    M, N, K, amn, bmn, sa, sb, ref = CASES[name]
    rng = np.random.default_rng(5)
    A = rng.normal(size=sa).astype(np.float32); B = rng.normal(size=sb).astype(np.float32)
    for layout, q in ((2, tf32), (3, bf16)):
        D = probe(J, M, N, K, amn, bmn, A, B, layout=layout)
        lanes, err = lane_map(D, ref(q(A), q(B)))
        print(name, "layout", layout, "rel err %.2e" % err, "|D|max %.3f" % np.abs(D).max(), "lanes", lanes[:4], lanes[16:20], flush=True)
