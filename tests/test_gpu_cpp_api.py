"""The C++ drop-in boundary on its own: a host program
that includes only include/janus/{schedule_gen,train}.hpp and links
libjanus_b200.so — no Python, no PyTorch — runs janus::train_step on
schedules from the reference-API generators.  Its losses equal the Python
binding's trainer on the same inputs bit for bit, and P stages equal one."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def demo(tmp_path_factory, built, has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")
    exe = str(tmp_path_factory.mktemp("cpp") / "train_step_demo")
    lib = os.path.join(ROOT, "paper_2605_18404_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tools", "cpp", "train_step_demo.cpp"), "-L" + lib, "-l:libjanus_b200.so",
                    "-Wl,-rpath," + lib, "-o", exe], check=True)
    return exe


def run_demo(exe, P, method, n_mb=4, steps=2, prec="tf32"):
    r = subprocess.run([exe, str(P), method, str(n_mb), str(steps), prec], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    return [l["loss"] for l in lines if "loss" in l], lines[-1]["block0_param_sum"], lines


@pytest.mark.parametrize("P,method", [(2, "symfold"), (2, "wavek"), (4, "hanayo"), (2, "onef1b")])
def test_cpp_train_step_matches_binding(janus, demo, P, method):
    losses, _, lines = run_demo(demo, P, method)
    assert all(np.isfinite(losses)) and losses[1] != losses[0]
    if method != "onef1b":  # folded layouts: P stages == one stage, bit for bit
        l1, s1, _ = run_demo(demo, 1, "symfold")
        assert losses == l1
    # the Python binding's trainer on the same synthetic inputs
    m = janus.Model(L=2, H=64, R=64, precision=janus.PREC_TF32)
    params = m.synth_params(7)
    bs = [janus.synth_batch(m, [32 + 4 * (i % 3)], 0.095, 100 + i, device_nl=True) for i in range(4)]
    meth = {"symfold": janus.METHOD_SYMFOLD, "wavek": janus.METHOD_WAVEK, "onef1b": janus.METHOD_ONEF1B,
            "hanayo": janus.METHOD_HANAYO}[method]
    t = janus.Trainer(m, params, P, meth, 4, k=min(4, 2 * P), max_atoms=64, max_edges=64 * 120, max_struct=1,
                      graphs=True, lanes=1)
    py = []
    for _ in range(2):
        t.load_many(bs)
        py.append(t.step(lr=1e-3).loss)
    t.close()
    if method == "onef1b":
        np.testing.assert_allclose(losses, py, rtol=1e-6)
    else:
        assert losses == py
