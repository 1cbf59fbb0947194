"""One rank of the same-GPU multi-process harness (tests/test_gpu_multirank.py).

Runs the per-rank (local_stages = 0) executor path exactly as a one-process-
per-GPU job does — its own trainer holding only this rank's blocks, channel
streams, blocking-rendezvous transfers and group all-reduces — but on the IPC
transport, so N processes can share the one GPU this run has.

  python tests/multirank_worker.py <json config> <rank> <out.npz>
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def batches_for(J, m, cfg, replica):
    n = cfg["n_mb"]
    return [J.synth_batch(m, cfg["atoms"][(replica * n + i) % len(cfg["atoms"])], 0.095, 100 + replica * n + i)
            for i in range(n)]


def run_rank(J, cfg, rank, comm, barrier=None):
    """One rank's whole job on an existing communicator: its own per-rank
    trainer (local=False), cfg["steps"] steps, then its blocks' parameters and
    reduced gradients."""
    P, D = cfg["P"], cfg["dp"]
    m = J.Model(L=cfg["L"], H=64, R=64, precision=J.PREC_TF32 if cfg["prec"] == "tf32" else J.PREC_FP32)
    params = m.synth_params(cfg["seed"])
    tr = J.Trainer(m, params, P, cfg["method"], cfg["n_mb"], k=cfg.get("k", 1), max_atoms=cfg["max_atoms"],
                   max_edges=cfg["max_atoms"] * 120, max_struct=2, local=False, comm=comm, rank=rank, device=0,
                   dp=D, lanes=cfg["lanes"])
    print(f"rank {rank}: trainer created", flush=True)
    bs = batches_for(J, m, cfg, rank // P)
    res = {}
    losses = []
    for step in range(cfg["steps"]):
        tr.load_many(bs)
        if barrier:  # thread ranks share one CUDA context: no rank may spin on a peer while another
            barrier()  # is still inside an allocating (possibly device-synchronising) call
        s = tr.step(lr=1e-3)
        losses.append(s.loss)
        print(f"rank {rank}: step {step} done", flush=True)
        res["p2p_bytes"] = s.p2p_bytes
    for b in range(P):
        for fr in (False, True):
            try:
                st = tr.stage(b, force_replica=fr)
            except J.JanusError:
                continue
            tag = f"{'F' if fr else 'E'}{b}"
            res[f"params_{tag}"] = st.params()
            res[f"grads_{tag}"] = st.grad_buffer()
    res["loss"] = np.array(losses)
    tr.close()
    return res


def run_threads(J, cfg, timeout):
    """All ranks as THREADS of this (fresh) process on the one GPU
    (Comm.threads): each builds its own per-rank trainer; ctypes releases the
    GIL, so the ranks issue concurrently.  Returns per-rank results or raises
    with every rank's error."""
    import tempfile
    import threading

    world = cfg["P"] * cfg["dp"]
    with tempfile.TemporaryDirectory() as d:
        res, errs = [None] * world, [None] * world
        bar = threading.Barrier(world)

        def one(r):
            try:
                comm = J.Comm.threads(d, world, r, 0)
                try:
                    res[r] = run_rank(J, cfg, r, comm, barrier=lambda: bar.wait(timeout))
                finally:
                    comm.close()
            except Exception as ex:  # noqa: BLE001
                errs[r] = ex
                print(f"rank {r} error: {ex!r}", file=sys.stderr, flush=True)

        ts = [threading.Thread(target=one, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        bad = [f"rank {r}: {e!r}" for r, e in enumerate(errs) if e is not None]
        if bad:
            raise RuntimeError("\n".join(bad))
        return res


def main():
    import faulthandler

    if int(os.environ.get("WORKER_DUMP", 0)) > 0:  # the harness's timeout: show where this rank is stuck
        faulthandler.dump_traceback_later(int(os.environ["WORKER_DUMP"]), exit=False)
    cfg = json.loads(sys.argv[1])
    import paper_2605_18404_b200 as J

    if sys.argv[2] == "threads":  # every rank as a thread of this process: out = prefix of per-rank files
        res = run_threads(J, cfg, int(os.environ.get("THREAD_BARRIER_TIMEOUT", 120)))
        for r, x in enumerate(res):
            np.savez(f"{sys.argv[3]}.{r}.npz", **x)
        return
    rank = int(sys.argv[2])
    out = sys.argv[3]
    comm = J.Comm.ipc(cfg["dir"], cfg["P"] * cfg["dp"], rank, 0)
    res = run_rank(J, cfg, rank, comm)
    comm.close()
    np.savez(out, **res)


if __name__ == "__main__":
    main()
