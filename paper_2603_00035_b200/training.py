"""Config C5 of SURVEY.md §8: learning Randers fields from covariates.

The paper's training workload: a small
CNN encoder maps covariates to raw field channels; the differentiable
projection layer makes them feasible; the eikonal solve produces arrival
times; an MSE on the observed (reached) nodes is the loss.  Gradients flow
back through the solve by the adjoint (torch_ops.EikonalSolve) and through
the projection by its VJP, then into the encoder.  Samples are independent,
so data parallelism is plain DDP over NCCL: the only collective is the
all-reduce of the encoder's gradients (~0.46 MB fp32), which DDP buckets and
overlaps with the backward.  The encoder is ordinary PyTorch (not the hot
path); the solve, adjoint and projection are the CUDA library.
"""
from __future__ import annotations

import contextlib

import torch
import torch.nn.functional as F

from . import torch_ops

# Encoder arithmetic.  "fp32": fp32 tensors with cuDNN's default math (torch
# allows TF32 for convolutions by default).  "bf16": bf16 autocast with
# channels-last activations (tensor-core convolutions).  The raw channels are
# cast to fp64 before the projection either way: the solver path is fp64.
ENCODER_PRECISIONS = ("fp32", "bf16")


def _check_precision(precision):
    if precision not in ENCODER_PRECISIONS:
        raise ValueError(f"encoder precision must be one of {ENCODER_PRECISIONS}, got {precision!r}")


def prepare_encoder(model, precision="fp32"):
    """Lay the encoder's weights out for `precision` (channels-last for bf16)."""
    _check_precision(precision)
    if precision == "bf16":
        model.to(memory_format=torch.channels_last)
    return model


def encoder_input(covariates, precision="fp32"):
    """Covariates (B, C, R, C) in the layout the encoder runs in."""
    _check_precision(precision)
    if precision == "bf16":
        return covariates.contiguous(memory_format=torch.channels_last)
    return covariates


def encoder_autocast(precision="fp32"):
    """Context the encoder's forward runs under."""
    _check_precision(precision)
    if precision == "bf16":
        return torch.autocast("cuda", dtype=torch.bfloat16)
    return contextlib.nullcontext()


class RandersEncoder(torch.nn.Module):
    """5-layer 3x3 CNN, 64 hidden channels (~116K parameters)."""

    def __init__(self, in_ch: int = 3, hidden: int = 64, layers: int = 5):
        super().__init__()
        chans = [in_ch] + [hidden] * (layers - 1) + [5]
        self.convs = torch.nn.ModuleList(
            torch.nn.Conv2d(a, b, 3, padding=1) for a, b in zip(chans[:-1], chans[1:]))

    def forward(self, x):
        for i, conv in enumerate(self.convs):
            x = conv(x)
            if i + 1 < len(self.convs):
                x = F.relu(x)
        return x


PROJECTION = dict(eps_min=0.5, lambda_max=2.5, tau=0.4, euclid_cap=10.0)


def raw_to_preprojection(raw):
    """Raw channels (B, 5, R, C) -> the fp64 parameters before the
    feasibility projection: an SPD parameterisation (softplus diagonal,
    bounded correlation) and a bounded drift."""
    raw = raw.to(torch.float64)
    g11 = F.softplus(raw[:, 0]) + 0.5
    g22 = F.softplus(raw[:, 2]) + 0.5
    g12 = 0.9 * torch.tanh(raw[:, 1]) * torch.sqrt(g11 * g22)
    b1, b2 = 0.5 * torch.tanh(raw[:, 3]), 0.5 * torch.tanh(raw[:, 4])
    return [x.contiguous() for x in (g11, g12, g22, b1, b2)]


def raw_to_fields(raw, eps_min=0.5, lambda_max=2.5, tau=0.4, euclid_cap=10.0):
    """Map raw channels (B, 5, R, C) to feasible fp64 Randers fields: the
    parameterisation followed by the exact, differentiable projection
    (project_spd then project_drift) as its own pass."""
    pre = raw_to_preprojection(raw)
    shp = pre[0].shape
    flat = [x.reshape(-1).contiguous() for x in pre]
    out = torch_ops.project(*flat, eps_min, lambda_max, tau, euclid_cap)
    return [x.reshape(shp) for x in out]


def c5_loss(model, covariates, sources, observed, targets, h, tol=1e-6, max_iters=50, precision="fp32",
            fused_projection=True):
    """Mean over the batch of 0.5 * sum of squared arrival-time errors on the
    observed, reached nodes (the data term of the paper's training loss).
    fused_projection: the feasibility projection runs inside the solver's load
    stage and its VJP inside the backward (torch_ops.projected_eikonal_solve,
    bitwise the same as the separate projection pass)."""
    with encoder_autocast(precision):
        raw = model(covariates)
    if fused_projection:
        pre = raw_to_preprojection(raw.contiguous())
        t = torch_ops.projected_eikonal_solve(*pre, sources, h, tol, max_iters, **PROJECTION)
    else:
        fields = raw_to_fields(raw.contiguous())
        t = torch_ops.eikonal_solve(*fields, sources, h, tol, max_iters)
    mask = observed.bool() & (t < 1e9)
    diff = torch.where(mask, t - targets, torch.zeros_like(t))
    return 0.5 * (diff * diff).sum() / t.shape[0]


def train_step(model, optimizer, batch, h, precision="fp32"):
    """One optimiser step on a batch (covariates, sources, observed, targets)."""
    optimizer.zero_grad(set_to_none=True)
    loss = c5_loss(model, *batch, h, precision=precision)
    loss.backward()
    optimizer.step()
    return loss.detach()
