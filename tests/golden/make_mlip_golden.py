"""Generate the golden vectors that pin the fp64 oracle (oracle/mlip_oracle.c).

The reference has no numeric implementation of the four-phase step
(SPEC.md:15), so the golden outputs come from PyTorch fp64 autograd
double-backward (tests/golden/torch_model.py) — the arithmetic engine the
paper's system used — on small seeded inputs.  The oracle is
then checked against these fixtures on every CPU test run, and the GPU path
against the oracle.  Usage: python tests/golden/make_mlip_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)

import oracle as O  # noqa: E402
import torch_model as T  # noqa: E402

CASES = [
    # name, model kwargs, cell sizes (atoms), box lengths, seed
    ("tiny", dict(L=2, H=8, R=8, r_c=3.0), [6], [4.0], 1),
    ("two_struct", dict(L=1, H=4, R=6, r_c=2.5), [5, 7], [3.2, 3.6], 2),
    ("deep_small_cell", dict(L=3, H=16, R=8, r_c=3.0), [9], [2.8], 3),  # cell < r_c: self images
]


def make_case(model, sizes, boxes, seed):
    rng = np.random.default_rng(seed)
    pos, sp, sid = [], [], []
    for s, (n, L) in enumerate(zip(sizes, boxes)):
        pos.append(rng.uniform(0, L, (n, 3)))
        sp.append(rng.integers(0, model.n_species, n))
        sid.append(np.full(n, s))
    N = sum(sizes)
    batch = O.Batch(np.concatenate(pos), np.concatenate(sp), np.concatenate(sid), boxes,
                    rng.normal(0, 1, len(sizes)), rng.normal(0, 0.1, (N, 3)))
    params = rng.normal(0, 0.3, model.param_count())
    return batch, params


def main():
    out = {}
    for name, kw, sizes, boxes, seed in CASES:
        model = O.Model(**kw)
        batch, params = make_case(model, sizes, boxes, seed)
        nl = O.build_nbrlist(model, batch)
        E, F, loss, grad = T.step(model, batch, nl, params)
        r = O.step(model, batch, nl, params)
        err = np.abs(r.grad - grad).max() / np.abs(grad).max()
        print(f"{name}: N={batch.n_atoms} E={nl.n_edges} loss={loss:.6f} oracle-vs-autograd grad relerr={err:.2e}")
        pre = f"{name}__"
        for k, v in dict(model=np.array([model.L, model.H, model.R, model.n_species], np.int64),
                         model_f=np.array([model.r_c, model.w_E, model.w_F]), pos=batch.pos,
                         species=batch.species, struct_id=batch.struct_id, cell=batch.cell,
                         E_target=batch.E_target, F_target=batch.F_target, params=params,
                         row_ptr=nl.row_ptr, col=nl.col, shift=nl.shift, rev=nl.rev,
                         E=E, F=F, loss=np.array([loss]), grad=grad).items():
            out[pre + k] = v
    path = os.path.join(HERE, "mlip_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
