#!/usr/bin/env python3
"""Device LM (nbrlist.cu) vs the host neighbour-list build, per micro-batch.

Times janus_nbrlist_build_device (wall clock around the call, which syncs its
stream once: the LM latency a load sees) and janus_nbrlist_build (host, one
thread) on the configs' cells; prints one JSON line per case.  Kernel shares:
run under `ncu --metrics gpu__time_duration.sum` (profiles/)."""
import ctypes
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_18404_b200 as J  # noqa: E402

CASES = [("C1 64-atom", [64], 0.095), ("C2 256-atom", [256], 0.095), ("C3 512-atom", [512], 0.095),
         ("C4 mixed 128..1024", [128, 250, 256, 432, 500, 512, 686, 864, 1000, 1024], 0.095),
         ("C5 4096-atom dense", [4096], 0.19),
         ("C2 x 32 micro-batches (one batched LM, the bench's e2e)", [256] * 32, 0.095)]


def main():
    rt = J.cudart()
    for name, sizes, rho in CASES:
        P, SID, C = [], [], []
        for s, n in enumerate(sizes):
            pos, sp, L, Et, Ft = J.synth_cell(n, rho, 4, 7000 + s)
            P.append(pos); SID.append(np.full(n, s, np.int32)); C.append(L)
        pos, sid, cell = np.concatenate(P), np.concatenate(SID), np.array(C)
        n = len(pos)
        max_edges = n * 200
        bufs = []
        for b in (pos.nbytes, sid.nbytes, 4 * (n + 1), 4 * max_edges, 12 * max_edges, 4 * max_edges):
            p = ctypes.c_void_p()
            assert rt.cudaMalloc(ctypes.byref(p), b) == 0
            bufs.append(p.value)
        rt.cudaMemcpy(bufs[0], pos.ctypes.data, pos.nbytes, 1)
        rt.cudaMemcpy(bufs[1], sid.ctypes.data, sid.nbytes, 1)
        h = ctypes.c_void_p()
        J.check(J.lib().janus_nbrlist_create(n, len(cell), max_edges, 0, ctypes.byref(h)))
        ne = ctypes.c_int32()
        call = lambda: J.check(J.lib().janus_nbrlist_build_device(  # noqa: E731
            h, n, len(cell), bufs[0], bufs[1], cell.ctypes.data_as(ctypes.c_void_p), 5.0, bufs[2], bufs[3],
            bufs[4], bufs[5], ctypes.byref(ne), None))
        for _ in range(5):
            call()
        iters = 50
        t0 = time.perf_counter()
        for _ in range(iters):
            call()
        dev_us = (time.perf_counter() - t0) / iters * 1e6
        E = ne.value
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < 1.0 or reps < 1:
            J.nbrlist(pos, sid, cell, 5.0, max_edges=max_edges)
            reps += 1
        host_us = (time.perf_counter() - t0) / reps * 1e6
        # compulsory bytes: pos + struct_id in, CSR out (row_ptr, col, shift, rev)
        alg = 24 * n + 4 * n + 4 * (n + 1) + 20 * E
        print(json.dumps({"case": name, "atoms": n, "edges": E, "device_us": dev_us, "host_us_1thread": host_us,
                          "speedup": host_us / dev_us, "alg_bytes": alg,
                          "alg_GBps_at_call_latency": alg / (dev_us * 1e-6) / 1e9}), flush=True)
        J.lib().janus_nbrlist_destroy(h)
        for p in bufs:
            rt.cudaFree(p)


if __name__ == "__main__":
    main()
