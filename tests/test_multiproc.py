"""N>1 host logic on CPU: two processes over torch.distributed (gloo,
127.0.0.1), as bench.py and the NCCL executor run one process per GPU.

* Cross-rank channel pairing.  NCCL pairs point-to-point messages in issue
  order per (communicator, peer), and the executor gives every flow its own
  communicator (executor.cpp, DepGraph channel key graph.hpp:95-97).  So for
  every (sender, receiver, flow) the sender's sequence of micro-batches must
  equal the receiver's.  Each rank extracts ITS device list from the generated
  schedule, the lists are exchanged with all_gather_object, and each rank
  checks the pairing against the other's list — the same invariant the
  executor asserts before it lets NCCL run.
* bench.py's reference arm under torchrun with 2 ranks: rank 0 alone runs and
  prints one JSON line; rank 1 exits 0 without work.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PAIR = {"SAE": "RAE", "SAF": "RAF", "SGF": "RGF", "SGE": "RGE"}


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def device_comms(text: str, dev: int):
    """Ordered (kind, mb, peer) comm instructions of device `dev`."""
    out = []
    for line in text.splitlines()[1:]:
        f = line.split()
        if not f or f[0] != f"D{dev}":
            continue
        kind = f[2]
        if kind[:2] in ("SA", "SG", "RA", "RG"):
            out.append((kind, int(f[3].split("=")[1]), int(f[5].split("=")[1])))
    return out


def _pairing_worker(rank: int, world: int, port: int, results):
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import paper_2605_18404_b200 as J

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        checked = 0
        for method, k in ((J.METHOD_SYMFOLD, 1), (J.METHOD_WAVEK, 2), (J.METHOD_WAVEK, 4)):
            for n_mb in (1, 4, 7):
                text = J.schedule_text(method, world, n_mb, min(k, n_mb))
                mine = device_comms(text, rank)
                lists = [None] * world
                dist.all_gather_object(lists, mine)
                for peer in range(world):
                    if peer == rank:
                        continue
                    for send, recv in PAIR.items():
                        sent = [mb for kind, mb, p in mine if kind == send and p == peer]
                        got = [mb for kind, mb, p in lists[peer] if kind == recv and p == rank]
                        assert sent == got, (method, n_mb, send, rank, peer, sent, got)
                        checked += len(sent)
                # every transfer of this rank has a partner
                n_send = sum(1 for kind, _, _ in mine if kind in PAIR)
                n_recv = sum(1 for kind, _, _ in mine if kind in PAIR.values())
                tot = [None] * world
                dist.all_gather_object(tot, (n_send, n_recv))
                assert sum(a for a, _ in tot) == sum(b for _, b in tot)
        results[rank] = checked
    finally:
        dist.destroy_process_group()


def test_channel_pairing_two_ranks(janus):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    mp.start_processes(_pairing_worker, args=(2, free_port(), results), nprocs=2, start_method="spawn", join=True)
    assert set(results.keys()) == {0, 1}
    assert results[0] > 0 and results[1] > 0


@pytest.mark.timeout(600)
def test_bench_reference_arm_torchrun_two_ranks(janus, oracle):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=580, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["value"] > 0 and d["unit"] == "structures/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0
