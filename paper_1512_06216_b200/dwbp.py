"""DWBP glue: drive libposeidon from PyTorch autograd (Alg. 2).

Every parameterised layer of a model becomes a Poseidon layer:

* FC layers (``nn.Linear``) that SACP assigns to SFB run through
  ``SFBLinearFunction``: backward computes only E_i = dX (the error message the
  layer below needs, Alg. 2 line 7) and hands the per-sample factors (grad_out,
  input) to ``poseidon_sync_fc_sfb`` — the local dW is never formed (Eq. 5).
* Other layers (conv, and FC layers the rule sends to PS) keep their
  parameters as views into one padded flat buffer per layer (W row-major then
  bias, ``poseidon_shard_range``), their ``.grad`` as views into a matching
  gradient buffer, and fire ``poseidon_backprop_hook`` from a
  post-accumulate-grad hook once all of the layer's gradients have landed.
* A forward pre-hook makes the next forward of layer i wait for layer i's sync
  (``poseidon_wait_layer``): the only synchronisation DWBP needs.
* With ``FLAG_SSP1`` (staleness s = 1, or 1..5 via ``Context.set_staleness``)
  the library applies a layer's update s hooks later; PS gradients then rotate
  through s + 1 arena buffers, so the parameters' ``.grad`` views are
  re-pointed after every iteration, and ``flush()`` applies the deferred
  updates.

All arithmetic of the sync happens in the library; this module only moves
pointers and streams.  The optimiser step IS the sync (SGD applied by K1/K2),
so there is no torch optimiser.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

import torch
import torch.nn as nn

from . import binding as B


@dataclass
class LayerPlan:
    layer_id: int
    name: str
    module: nn.Module
    kind: int
    M: int
    N: int
    K: int
    scheme: int
    rule_scheme: int
    costs: tuple
    n: int = 0
    padded: int = 0
    flat_w: Optional[torch.Tensor] = None
    flat_g: Optional[torch.Tensor] = None
    pending: int = 0
    n_params: int = 0
    hook_handles: List = field(default_factory=list)


def _view_like(seg: torch.Tensor, p: torch.Tensor) -> torch.Tensor:
    """View a flat buffer segment with p's shape AND memory format (a channels_last conv weight
    keeps its NHWC strides, so cuDNN sees no layout change; the PS sync is elementwise over the
    flat buffer and does not care about the element order)."""
    if p.dim() == 4 and not p.is_contiguous() and p.is_contiguous(memory_format=torch.channels_last):
        o, i, h, w = p.shape
        return seg.view(o, h, w, i).permute(0, 3, 1, 2)
    return seg.view_as(p)


class SFBLinearFunction(torch.autograd.Function):
    """y = x W^T + b; backward returns dX only and triggers the SFB sync."""

    @staticmethod
    def forward(ctx, x, weight, bias, plan, sync, post_input):
        if x.dim() != 2 or x.shape[0] != plan.K or x.shape[1] != plan.N:
            # the sufficient factors are K x N inputs and K x M error messages with the K the layer was
            # registered with: a partial batch or a >2-D input would be misread by the library
            raise ValueError(f"SFB layer {plan.name}: input must be ({plan.K}, {plan.N}) (registered per-GPU "
                             f"batch K, in_features), got {tuple(x.shape)}")
        if post_input:
            # FLAG_EARLY_V: the input factors V = a_i are final now; their broadcast overlaps the rest of
            # the forward and the backward (the hook then moves only U)
            sync.ctx.sfb_post_input(plan.layer_id, x.contiguous(), torch.cuda.current_stream())
        ctx.save_for_backward(x, weight)
        ctx.plan = plan
        ctx.sync = sync
        ctx.bias = bias
        if bias is not None:
            return torch.addmm(bias, x, weight.t())
        return x @ weight.t()

    @staticmethod
    def backward(ctx, grad_out):
        x, weight = ctx.saved_tensors
        grad_out = grad_out.contiguous()
        # E_i for the layer below (Alg. 2 line 7) BEFORE "Communicate" (line 9): the in-place
        # update of W on the library's stream is ordered after this read by the ready event.
        grad_x = grad_out @ weight if ctx.needs_input_grad[0] else None
        ctx.sync.sfb_backward(ctx.plan, grad_out, x.contiguous(), weight, ctx.bias)
        return grad_x, None, None, None, None, None


class PoseidonSync:
    """Registers a model's layers with a libposeidon context and installs the
    DWBP hooks.  ``K`` is the per-GPU batch (number of sufficient-factor pairs
    per worker per FC layer)."""

    def __init__(self, model: nn.Module, ctx: B.Context, K: int, lr: float,
                 scheme: str = "auto", recon: int = B.RECON_TF32, arena: bool = False, bucket_bytes: int = 0,
                 overrides: Optional[Dict[str, str]] = None):
        self.model = model
        self.ctx = ctx
        self.K = K
        self.lr = float(lr)
        self.plans: List[LayerPlan] = []
        self.by_module: Dict[nn.Module, LayerPlan] = {}
        ctx.set_lr(self.lr)
        self.ssp = bool(getattr(ctx, "flags", 0) & B.FLAG_SSP1)
        self.early_v = bool(getattr(ctx, "flags", 0) & B.FLAG_EARLY_V)
        # FLAG_INPLACE_FACTORS: the library reads grad_out and x where they are, on its own streams (K1 at
        # world 1, else the pack before the factor broadcast), so their memory must not be handed out again
        # before the sync is done.  The glue holds the two tensors until the layer's next forward has waited
        # for the sync (poseidon_wait_layer in the pre-forward hook) and only then drops them: the allocator
        # then reuses the blocks on the compute stream, already ordered after the sync.  (record_stream on the
        # library's streams did the same job but made the caching allocator defer and re-allocate blocks: 1 in
        # ~5 C3 runs lost half its images/s, profiles/r2/factors_r2.md.)
        self.hold_factors = bool(getattr(ctx, "flags", 0) & B.FLAG_INPLACE_FACTORS) and not self.ssp and \
            not (getattr(ctx, "flags", 0) & B.FLAG_DWBP_OFF)
        self.held: Dict[int, tuple] = {}
        if self.ssp and not arena:
            raise ValueError("FLAG_SSP1 needs the library arena (arena=True): PS gradients are double-buffered")
        self.arena = arena
        self.nvls_active = False
        # overrides: layer name -> "auto" / "ps" / "sfb" / "sfps" for that layer only (e.g. the P >= 6 schedule
        # of C3, fc8 on the server, exercised at fewer GPUs)
        overrides = dict(overrides or {})
        layer_id = 0
        for name, mod in model.named_modules():
            if isinstance(mod, (nn.Linear, nn.Conv2d)):
                self._register(layer_id, name, mod, overrides.pop(name, scheme), recon)
                layer_id += 1
        if overrides:
            raise ValueError(f"scheme overrides for unknown layers: {sorted(overrides)}")
        if arena:
            # one library-owned gradient/parameter arena for all PS layers (symmetric NCCL windows
            # with FLAG_NVLS_PS: each PS sync is then one fused multimem kernel); optionally runs of
            # small PS layers sync as one bucket
            if bucket_bytes:
                ctx.set_ps_buckets(bucket_bytes)
            self.nvls_active = ctx.ps_arena()
            for plan in self.plans:
                if plan.scheme == B.SCHEME_PS:
                    self._bind_arena(plan)

    # ------------------------------------------------------------ setup ----
    def _register(self, lid, name, mod, scheme, recon):
        if isinstance(mod, nn.Linear):
            kind, M, N = B.LAYER_FC, mod.out_features, mod.in_features
        else:
            kind = B.LAYER_CONV
            M = mod.out_channels
            N = mod.weight[0].numel()  # in_channels/groups * kh * kw
        rule, costs = B.choose_scheme(kind, M, N, self.K, self.ctx.world)
        override = -1
        if scheme == "ps":
            override = B.SCHEME_PS
        elif scheme == "sfb" and kind == B.LAYER_FC:
            override = B.SCHEME_SFB
        elif scheme == "sfps" and kind == B.LAYER_FC:
            override = B.SCHEME_SFPS
        has_bias = mod.bias is not None
        chosen = self.ctx.register_layer(lid, kind, M, N, self.K, has_bias, override)
        plan = LayerPlan(lid, name, mod, kind, M, N, self.K, chosen, rule, costs)
        self.plans.append(plan)
        self.by_module[mod] = plan
        if chosen in (B.SCHEME_SFB, B.SCHEME_SFPS):   # factor schemes: the local dW is never formed
            self.ctx.set_recon(recon, lid)
            mod.weight.data = mod.weight.data.contiguous()
            self.ctx.bind_sfb_params(lid, mod.weight, mod.bias)
            self._wrap_linear(mod, plan)
        else:
            self._flatten_ps(mod, plan)
        h = mod.register_forward_pre_hook(self._pre_forward(plan))
        plan.hook_handles.append(h)

    def _point_grads(self, plan, gptr):
        """Make the layer's parameter gradients views of the arena gradient buffer at gptr."""
        mod = plan.module
        params = [mod.weight] + ([mod.bias] if mod.bias is not None else [])
        flat_g = B.device_view(gptr, (plan.padded,))
        off = 0
        for p in params:
            k = p.numel()
            p.grad = _view_like(flat_g[off:off + k], p)
            off += k
        plan.flat_g = flat_g

    def _bind_arena(self, plan):
        mod = plan.module
        params = [mod.weight] + ([mod.bias] if mod.bias is not None else [])
        gptr, wptr, padded = self.ctx.ps_layer_buffers(plan.layer_id)
        flat_g = B.device_view(gptr, (padded,))
        flat_w = B.device_view(wptr, (padded,))
        off = 0
        for p in params:
            k = p.numel()
            wv = _view_like(flat_w[off:off + k], p)
            wv.copy_(p.data)
            p.data = wv
            p.grad = _view_like(flat_g[off:off + k], p)
            off += k
        torch.cuda.synchronize()
        plan.flat_w, plan.flat_g, plan.padded = flat_w, flat_g, padded

    def _flatten_ps(self, mod, plan):
        params = [mod.weight] + ([mod.bias] if mod.bias is not None else [])
        n = sum(p.numel() for p in params)
        plan.n = n
        plan.n_params = len(params)
        for p in params:
            plan.hook_handles.append(p.register_post_accumulate_grad_hook(self._post_accumulate(plan)))
        if self.arena:
            return  # buffers come from the library arena after all layers are registered
        _, _, padded = B.shard_range(n, self.ctx.world, self.ctx.rank)
        dev = mod.weight.device
        flat_w = torch.zeros(padded, device=dev, dtype=torch.float32)
        flat_g = torch.zeros(padded, device=dev, dtype=torch.float32)
        off = 0
        for p in params:
            k = p.numel()
            wv = _view_like(flat_w[off:off + k], p)
            wv.copy_(p.data)
            p.data = wv
            p.grad = _view_like(flat_g[off:off + k], p)
            off += k
        plan.padded, plan.flat_w, plan.flat_g = padded, flat_w, flat_g
        self.ctx.bind_ps_buffers(plan.layer_id, flat_g, flat_w, n, B.PS_ZERO_GRAD)

    def _wrap_linear(self, mod, plan):
        sync = self

        def forward(x):
            # grad mode is read HERE (autograd runs Function.forward under no_grad): a forward that will
            # not be backpropagated (evaluation) posts no inputs
            post = sync.early_v and plan.scheme == B.SCHEME_SFB and torch.is_grad_enabled()
            return SFBLinearFunction.apply(x, mod.weight, mod.bias, plan, sync, post)

        mod.forward = forward

    # ------------------------------------------------------------ hooks ----
    def _pre_forward(self, plan):
        def hook(_mod, _inp):
            self.ctx.wait_layer(plan.layer_id, torch.cuda.current_stream())
            # the stream is ordered after the layer's sync now: its factors may be released
            getattr(self, "held", {}).pop(plan.layer_id, None)
        return hook

    def _post_accumulate(self, plan):
        def hook(_p):
            plan.pending += 1
            if plan.pending == plan.n_params:
                plan.pending = 0
                self.ctx.backprop_hook(plan.layer_id, torch.cuda.current_stream())
        return hook

    def sfb_backward(self, plan, grad_out, x, weight, bias):
        self.ctx.sync_fc_sfb(plan.layer_id, grad_out, x, weight, bias, self.lr, torch.cuda.current_stream())
        if getattr(self, "hold_factors", False):
            self.held[plan.layer_id] = (grad_out, x)

    # ------------------------------------------------------------ driver ----
    def iteration_end(self, stats: bool = False):
        out = self.ctx.iteration_end(torch.cuda.current_stream(), stats=stats)
        if self.ssp:
            # the next backward accumulates into the next of the s + 1 gradient buffers (zeroed by the
            # library before the next forward of the layer may start: poseidon_wait_layer orders it)
            for plan in self.plans:
                if plan.scheme == B.SCHEME_PS:
                    gptr = self.ctx.ps_layer_buffers(plan.layer_id)[0]
                    if gptr != plan.flat_g.data_ptr():
                        self._point_grads(plan, gptr)
        return out

    def flush(self, stream=None):
        """SSP: apply every deferred update (the last s iterations' syncs) on every rank, then order
        the stream after them (no-op for BSP)."""
        s = stream or torch.cuda.current_stream()
        self.ctx.flush(s)
        self.wait_all(s)

    def wait_all(self, stream=None):
        s = stream or torch.cuda.current_stream()
        for p in self.plans:
            self.ctx.wait_layer(p.layer_id, s)
        getattr(self, "held", {}).clear()   # ordered after every sync: the held factors may go

    def describe(self):
        out = []
        for p in self.plans:
            mpick, t_sfb, t_ps = B.choose_scheme_model(p.kind, p.M, p.N, p.K, self.ctx.world)
            m3, _, _, t_sfps = B.choose_scheme_model3(p.kind, p.M, p.N, p.K, self.ctx.world)
            out.append({"id": p.layer_id, "name": p.name, "kind": "fc" if p.kind == B.LAYER_FC else "conv",
                        "M": p.M, "N": p.N, "K": p.K,
                        "scheme": {B.SCHEME_SFB: "SFB", B.SCHEME_SFPS: "SFPS"}.get(p.scheme, "PS"),
                        "rule": "SFB" if p.rule_scheme == B.SCHEME_SFB else "PS",
                        "model": "SFB" if mpick == B.SCHEME_SFB else "PS",
                        "model3": {B.SCHEME_SFB: "SFB", B.SCHEME_SFPS: "SFPS"}.get(m3, "PS"),
                        "model_t_sfb_us": round(t_sfb, 1), "model_t_ps_us": round(t_ps, 1),
                        "model_t_sfps_us": round(t_sfps, 1),
                        "cost_sfb": p.costs[0], "cost_sf_ps": p.costs[1], "cost_full_ps": p.costs[2]})
        return out
