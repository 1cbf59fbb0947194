"""The per-rank (one process per GPU) executor path, run for real on ONE GPU
(VERDICT r01 item 2).

N processes share the GPU through the IPC transport (csrc/transport.hpp),
which has NCCL's blocking-rendezvous semantics: a send cannot complete before
its receive is posted, collectives need every member.  Each process builds
its own trainer with local_stages = 0 — only its own blocks, per-channel
communicators and streams, mirror transfers and group all-reduces — exactly
the code an 8-GPU job runs over NCCL.  Checks:

* SymFold / WaveK / Hanayo-2nd at P = 2 and 4 and 1F1B-2nd at P = 2 and 4:
  parameters and reduced gradients after two steps are BIT-IDENTICAL to the
  single-process local mode (same lanes => same kernel grids), and the loss
  sums match;
* PP x DP 2 x 2 (dp_degree = 2): each replica runs its own micro-batches, the
  stage replicas all-reduce before OS; parameters match the local-mode run of
  all micro-batches within fp32 re-association error (the replica sums are
  added in a different order than the micro-batch-ordered ledger);
* bench.py --gpus 2 under torchrun on the IPC transport prints its line;
* the same per-rank path with the ranks as threads of one process
  (Comm.threads), and the trainer's refusal to run peer-blocking streams on
  shared hardware queues.

Two process-wide CUDA settings are required for any peer-blocking path
(NCCL's too) and are set by conftest.py: CUDA_MODULE_LOADING=EAGER (a
lazily loaded kernel's first launch can wait behind a kernel blocked on a
peer) and CUDA_DEVICE_MAX_CONNECTIONS >= the rank's streams.
"""
import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import multirank_worker as W  # noqa: E402


def run_ranks_threads(cfg, timeout=int(os.environ.get("MULTIRANK_TIMEOUT", 420))):
    """All ranks as THREADS of one process on the one GPU (Comm.threads).  The
    process is a fresh one (tests/multirank_worker.py threads): the ranks share
    its CUDA context, and CUDA maps streams to hardware queues in creation
    order over the context's life, so a long-lived test process could make
    two live peer-blocking streams share a queue.  A rank that hangs ends the
    worker after `timeout` s with the executor's hang report."""
    world = cfg["P"] * cfg["dp"]
    with tempfile.TemporaryDirectory() as d:
        prefix = os.path.join(d, "out")
        env = dict(os.environ, JANUS_HANG_REPORT=str(max(5, timeout - 25)), THREAD_BARRIER_TIMEOUT=str(min(120, timeout)))
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "multirank_worker.py"), json.dumps(cfg), "threads",
                            prefix], cwd=ROOT, capture_output=True, text=True, timeout=timeout + 30, env=env)
        assert r.returncode == 0, (r.stdout[-2000:] + r.stderr[-4000:])
        return [dict(np.load(f"{prefix}.{q}.npz")) for q in range(world)]


def run_ranks(cfg, timeout=int(os.environ.get("MULTIRANK_TIMEOUT", 420))):
    """All ranks as separate PROCESSES on the one GPU (Comm.ipc, CUDA-IPC
    regions; the contexts are time-sliced).  The env of conftest.py (eager
    kernel loading, a hardware queue per stream) is inherited."""
    world = cfg["P"] * cfg["dp"]
    with tempfile.TemporaryDirectory() as d:
        cfg = dict(cfg, dir=d)
        procs, outs, logs = [], [], []
        env = dict(os.environ, WORKER_DUMP=str(max(10, timeout - 15)),  # python stacks before the kill
                   JANUS_HANG_REPORT=str(max(5, timeout - 25)))  # and the unfinished instructions
        for r in range(world):
            out = os.path.join(d, f"out{r}.npz")
            outs.append(out)
            logs.append(open(os.path.join(d, f"log{r}.txt"), "w+"))
            procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "multirank_worker.py"),
                                           json.dumps(cfg), str(r), out], cwd=ROOT, stdout=logs[-1],
                                          stderr=subprocess.STDOUT, text=True, start_new_session=True, env=env))
        timed_out = False
        try:
            for p in procs:
                p.wait(timeout=timeout)
        except subprocess.TimeoutExpired:
            timed_out = True
        finally:
            for p in procs:
                if p.poll() is None:
                    os.killpg(p.pid, 9)
                    p.wait()
        texts = []
        for f in logs:
            f.seek(0)
            texts.append(f.read())
            f.close()
        for r, p in enumerate(procs):
            assert p.returncode == 0, f"rank {r} failed{' (timeout)' if timed_out else ''}:\n" + \
                "\n".join(f"--- rank {q}\n{t[-2500:]}" for q, t in enumerate(texts))
        return [dict(np.load(o)) for o in outs]


def run_local(janus, cfg, n_mb_total=None):
    m = janus.Model(L=cfg["L"], H=64, R=64, precision=janus.PREC_TF32 if cfg["prec"] == "tf32" else janus.PREC_FP32)
    params = m.synth_params(cfg["seed"])
    bs = []
    for r in range(cfg["dp"]):
        bs += W.batches_for(janus, m, cfg, r)
    tr = janus.Trainer(m, params, cfg["P"], cfg["method"], len(bs), k=cfg.get("k", 1), max_atoms=cfg["max_atoms"],
                       max_edges=cfg["max_atoms"] * 120, max_struct=2, local=True, lanes=cfg["lanes"])
    losses = []
    for _ in range(cfg["steps"]):
        tr.load_many(bs)
        losses.append(tr.step(lr=1e-3).loss)
    res = {}
    for b in range(cfg["P"]):
        res[f"params_E{b}"] = tr.stage(b).params()
        res[f"grads_E{b}"] = tr.stage(b).grad_buffer()
    tr.close()
    return res, losses


def gather(ranks, key):
    for r in ranks:
        if key in r:
            return r[key]
    raise KeyError(key)


BASE = dict(L=2, n_mb=4, atoms=[[32], [40], [27], [36]], max_atoms=64, seed=21, steps=2, prec="fp32", lanes=2, dp=1)


@pytest.fixture(scope="module")
def gpu(has_gpu):
    if not has_gpu:
        pytest.skip("no GPU")


@pytest.mark.parametrize("P,method,k,prec", [(2, 0, 1, "fp32"), (4, 0, 1, "fp32"), (2, 1, 4, "fp32"), (4, 1, 4, "tf32"),
                                             (4, 4, 1, "fp32"), (2, 2, 1, "fp32"), (4, 2, 1, "fp32")])
def test_per_rank_bit_identical_to_local(janus, gpu, P, method, k, prec):
    cfg = dict(BASE, P=P, method=method, k=k, prec=prec)
    ranks = run_ranks(cfg)
    ref, ref_loss = run_local(janus, cfg)
    for b in range(P):
        assert np.array_equal(gather(ranks, f"params_E{b}"), ref[f"params_E{b}"]), f"block {b} params"
        assert np.array_equal(gather(ranks, f"grads_E{b}"), ref[f"grads_E{b}"]), f"block {b} grads"
        if method == 2:  # 1F1B-2nd: the force replica took the same step on the all-reduced gradient
            assert np.array_equal(gather(ranks, f"params_F{b}"), ref[f"params_E{b}"])
    loss = np.sum([r["loss"] for r in ranks], axis=0)
    np.testing.assert_allclose(loss, ref_loss, rtol=1e-6)
    assert all(r["p2p_bytes"] > 0 for r in ranks)


@pytest.mark.parametrize("method", [0, 1])
def test_pp_dp_2x2(janus, gpu, method):
    cfg = dict(BASE, P=2, dp=2, method=method, k=2, n_mb=2)
    ranks = run_ranks(cfg)
    ref, ref_loss = run_local(janus, cfg)  # all 4 micro-batches through one 2-stage pipeline
    for b in range(2):
        for rep in range(2):  # both replicas of the stage hold the same all-reduced gradient and parameters
            rr = ranks[rep * 2 + b]
            g_ref = ref[f"grads_E{b}"]
            assert np.abs(rr[f"grads_E{b}"] - g_ref).max() <= 1e-6 * np.abs(g_ref).max()
            assert np.abs(rr[f"params_E{b}"] - ref[f"params_E{b}"]).max() < 1e-6
        assert np.array_equal(ranks[b][f"params_E{b}"], ranks[2 + b][f"params_E{b}"])
    loss = np.sum([r["loss"] for r in ranks], axis=0)
    np.testing.assert_allclose(loss, ref_loss, rtol=1e-5)


@pytest.mark.parametrize("P,method,k", [(2, 0, 1), (2, 1, 2), (2, 2, 1)])
def test_thread_ranks_bit_identical_to_local(janus, gpu, P, method, k):
    """The same per-rank path with the ranks as threads of one process
    (Comm.threads: one CUDA context, the ranks' kernels run concurrently).
    All ranks' streams share the context's hardware queues, so only P=2 fits
    (P=4 is refused: test_thread_ranks_share_hardware_queues)."""
    cfg = dict(BASE, P=P, method=method, k=k)
    ranks = run_ranks_threads(cfg)
    ref, ref_loss = run_local(janus, cfg)
    for b in range(P):
        assert np.array_equal(gather(ranks, f"params_E{b}"), ref[f"params_E{b}"]), f"block {b} params"
        assert np.array_equal(gather(ranks, f"grads_E{b}"), ref[f"grads_E{b}"]), f"block {b} grads"
    np.testing.assert_allclose(np.sum([r["loss"] for r in ranks], axis=0), ref_loss, rtol=1e-6)


def test_thread_ranks_share_hardware_queues(janus, gpu):
    """Four ranks as threads of one process need more streams than the
    context's 32 hardware queues: refused at create (a peer-blocked stream
    would stall the unrelated streams sharing its queue — measured: a hang)."""
    cfg = dict(BASE, P=4, method=1, k=4)
    env = dict(os.environ, THREAD_BARRIER_TIMEOUT="20")
    try:  # the refused rank reports at create; its peers then give up at the barrier (or hang in teardown)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "multirank_worker.py"), json.dumps(cfg), "threads",
                            "/tmp/unused"], cwd=ROOT, capture_output=True, text=True, timeout=60, env=env)
        out = r.stdout + r.stderr
        assert r.returncode != 0
    except subprocess.TimeoutExpired as ex:
        out = "".join(x.decode(errors="replace") if isinstance(x, bytes) else (x or "") for x in (ex.stdout, ex.stderr))
    assert "ranks of this process" in out, out[-3000:]


def test_per_rank_runtime_checks(janus, gpu):
    """Per-rank mode refuses a process whose streams would share hardware
    queues (a peer-blocked stream could stall the stream its peer waits for)."""
    cfg = dict(BASE, P=2, method=0, k=1, lanes=40)
    with pytest.raises(AssertionError, match="CUDA_DEVICE_MAX_CONNECTIONS"):
        run_ranks_threads(cfg, timeout=60)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(900)
def test_bench_two_ranks_on_ipc(gpu):
    """bench.py's N>1 logic end to end (torchrun, 2 ranks, WaveK P=2) on the
    IPC transport: rank 0 prints one line with max-over-ranks timing."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--transport", "ipc", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=850)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["p2p_bytes_per_step"] > 0
    assert d["config"]["transport"] == "ipc (2 processes on one GPU)"
    assert d["roofline"] and "error" not in d["roofline"]
