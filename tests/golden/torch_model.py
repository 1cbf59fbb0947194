"""tests/golden/torch_model.py — TEST INFRASTRUCTURE: the canonical MLIP
 written directly in PyTorch fp64 so that autograd's
double-backward (create_graph=True, the arithmetic the paper's system used,
PAPER.md:494) produces an independent reference for E, F = -dE/dx, the loss
and dL/dtheta.  Used only to generate/verify the golden fixtures that pin the
C oracle (oracle/mlip_oracle.c); never imported by the product.
"""
from __future__ import annotations

import math

import torch


def unpack(model, params: torch.Tensor):
    """Split the flat parameter vector (layout in oracle/mlip_oracle.h)."""
    H, R, S, L = model.H, model.R, model.n_species, model.L
    out, off = {}, 0

    def take(name, *shape):
        nonlocal off
        n = 1
        for s in shape:
            n *= s
        out[name] = params[off:off + n].reshape(*shape)
        off += n

    take("Emb", S, H)
    for l in range(L):
        take(f"A{l}", R, H); take(f"alpha{l}", H); take(f"B{l}", H, H); take(f"beta{l}", H); take(f"W{l}", H, H)
        take(f"U{l}", H, H); take(f"ups{l}", H); take(f"V{l}", H, H)
    take("O", H, H); take("o", H); take("omega", H); take("bias", S)
    assert off == params.numel()
    return out


def energy(model, pos, species, struct_id, cell, n_struct, row, col, shift, P):
    """E_s for every structure; differentiable w.r.t. pos and P."""
    H, R, rc = model.H, model.R, model.r_c
    cell_e = cell[struct_id[row]]
    r = pos[col] + shift.to(pos.dtype) * cell_e[:, None] - pos[row]
    d = torch.sqrt((r * r).sum(-1))
    delta = rc / (R - 1)
    gamma = 1.0 / (2 * delta * delta)
    mu = torch.arange(R, dtype=pos.dtype) * delta
    phi = torch.exp(-gamma * (d[:, None] - mu[None, :]) ** 2)
    c = 0.5 * (torch.cos(math.pi * d / rc) + 1.0)
    silu = torch.nn.functional.silu
    h = P["Emb"][species]
    N = pos.shape[0]
    for l in range(model.L):
        z = phi @ P[f"A{l}"] + P[f"alpha{l}"]
        w = c[:, None] * (silu(z) @ P[f"B{l}"] + P[f"beta{l}"])
        v = h @ P[f"W{l}"]
        m = torch.zeros(N, H, dtype=pos.dtype).index_add(0, row, w * v[col])
        h = h + silu(m @ P[f"U{l}"] + P[f"ups{l}"]) @ P[f"V{l}"]
    t = h @ P["O"] + P["o"]
    e = silu(t) @ P["omega"] + P["bias"][species]
    return torch.zeros(n_struct, dtype=pos.dtype).index_add(0, struct_id, e)


def step(model, batch, nl, params_np):
    """Autograd double-backward: returns E, F, loss, grad as numpy."""
    dt = torch.float64
    pos = torch.tensor(batch.pos, dtype=dt, requires_grad=True)
    P_flat = torch.tensor(params_np, dtype=dt, requires_grad=True)
    P = unpack(model, P_flat)
    species = torch.tensor(batch.species, dtype=torch.long)
    sid = torch.tensor(batch.struct_id, dtype=torch.long)
    cell = torch.tensor(batch.cell, dtype=dt)
    row = torch.repeat_interleave(torch.arange(batch.n_atoms), torch.tensor(nl.row_ptr[1:] - nl.row_ptr[:-1], dtype=torch.long))
    col = torch.tensor(nl.col, dtype=torch.long)
    shift = torch.tensor(nl.shift, dtype=torch.long)
    E = energy(model, pos, species, sid, cell, batch.n_struct, row, col, shift, P)
    (dEdx,) = torch.autograd.grad(E.sum(), pos, create_graph=True)
    F = -dEdx
    Et = torch.tensor(batch.E_target, dtype=dt)
    Ft = torch.tensor(batch.F_target, dtype=dt)
    loss = model.w_E * ((E - Et) ** 2).sum() + model.w_F * ((F - Ft) ** 2).sum()
    (grad,) = torch.autograd.grad(loss, P_flat)
    return E.detach().numpy(), F.detach().numpy(), float(loss.detach()), grad.numpy()
