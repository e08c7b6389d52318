"""Whole-step parity against the oracle for a model trained through PoseidonSync (test infrastructure).

StepCapture records, for one training iteration, what each layer hands to the library: the sufficient
factors (grad_out, input) of SFB / SF-PS layers and the flat gradient (W row-major, then bias) of PS
layers at the moment the DWBP hook fires.  oracle_check() then recomputes every layer's synchronous
update with the fp64 oracle from the captures of ALL ranks -- O4 (sampled rows for big layers) for factor
layers, O6 (every element) for PS layers -- and gates W' with the Z13 metric (tests/parity.py).

safe_lr() picks a learning rate that makes every parameter's update at least ~1/4 of its magnitude, so the
fp32 gate is not dominated by the storage rounding of W' (reading Z13b).
"""
import numpy as np

import oracle as O
from parity import check_update

FACTOR_SCHEMES = (1, 2)   # SCHEME_SFB, SCHEME_SFPS


def _np(t):
    return t.detach().float().cpu().numpy()


def flat_params(mod):
    parts = [_np(mod.weight).reshape(-1)]
    if mod.bias is not None:
        parts.append(_np(mod.bias).reshape(-1))
    return np.concatenate(parts).astype(np.float64)


class StepCapture:
    def __init__(self, sync):
        self.sync = sync
        self.factors, self.grads = {}, {}
        self.plans = {p.name: p for p in sync.plans}
        by_id = {p.layer_id: p for p in sync.plans}
        orig_sfb = sync.sfb_backward

        def sfb(plan, grad_out, x, weight, bias):
            self.factors[plan.name] = (grad_out.detach().clone(), x.detach().clone())
            orig_sfb(plan, grad_out, x, weight, bias)

        sync.sfb_backward = sfb
        ctx = sync.ctx
        orig_hook = ctx.backprop_hook

        def hook(layer_id, stream=None):
            plan = by_id[layer_id]
            if plan.scheme not in FACTOR_SCHEMES:
                m = plan.module
                g = [m.weight.grad.detach().reshape(-1)]
                if m.bias is not None:
                    g.append(m.bias.grad.detach().reshape(-1))
                import torch
                self.grads[plan.name] = torch.cat(g).clone()
            orig_hook(layer_id, stream)

        ctx.backprop_hook = hook

    def snapshot(self):
        """Parameters before the iteration (call before the forward)."""
        self.before = {n: (_np(p.module.weight), None if p.module.bias is None else _np(p.module.bias))
                       for n, p in self.plans.items()}
        self.factors, self.grads = {}, {}


def gather_all(t, world):
    """Every rank's copy of a device tensor (world 1: just this one)."""
    if world == 1:
        return [t]
    import torch
    import torch.distributed as dist
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous())
    return parts


def oracle_check(cap, lr, world, tf32_tol=2e-3, max_rows=48, seed=0, names=None):
    """Recompute each layer's update with the oracle from every rank's captures and gate W'
    (tf32_tol: the gate of the factor layers' reconstruction, 1e-5 for the fp32 kernel K1r).
    Returns {layer name: update error}."""
    rng = np.random.default_rng(seed)
    errs = {}
    for name, plan in cap.plans.items():
        if names is not None and name not in names:
            continue
        mod = plan.module
        W0, b0 = cap.before[name]
        if plan.scheme in FACTOR_SCHEMES:
            G, X = cap.factors[name]
            Us = [_np(t) for t in gather_all(G, world)]
            Vs = [_np(t) for t in gather_all(X, world)]
            M = W0.shape[0]
            W0 = W0.reshape(M, -1)
            rows = np.arange(M) if M <= max_rows else \
                np.unique(np.concatenate([[0, M - 1], rng.integers(0, M, max_rows)]))
            Wr, br = O.sync_step_rows(W0[rows], None if b0 is None else b0[rows], Us, Vs, lr, rows)
            W1 = _np(mod.weight).reshape(M, -1)
            errs[name] = check_update(W0[rows], W1[rows], Wr, tf32_tol, f"{name} W (O4)")
            if b0 is not None:
                check_update(b0[rows], _np(mod.bias)[rows], br, 1e-5, f"{name} bias (O4)")
        else:
            grads = [_np(t).astype(np.float64) for t in gather_all(cap.grads[name], world)]
            w0 = np.concatenate([W0.reshape(-1)] + ([] if b0 is None else [b0.reshape(-1)])).astype(np.float64)
            ref = O.ps_step_flat(w0, grads, lr)
            errs[name] = check_update(w0, flat_params(mod), ref, 1e-5, f"{name} (O6)")
    return errs


def safe_lr(model, loss_fn, world=1):
    """max over parameters of max|p| / (4 max|grad p|) from a plain torch backward of loss_fn(model)
    (before any Poseidon hook exists); the max over ranks, so every rank uses the same lr."""
    import torch
    loss_fn(model).backward()
    lr = max(float(p.detach().abs().max() / (4 * p.grad.abs().max().clamp_min(1e-30))) for p in model.parameters())
    model.zero_grad(set_to_none=True)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([lr], device=next(model.parameters()).device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        lr = float(t.item())
    return lr
