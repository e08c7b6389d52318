"""Thin ctypes binding of libposeidon.so (include/poseidon.h).

Argument marshalling only: tensors become device pointers, streams become
cudaStream_t handles, status codes become PoseidonError.  Every step of the
sync path runs inside the library's CUDA kernels and NCCL calls; there is no
Python or CPU fallback — if the shared library is missing this module raises
at import time.
"""
from __future__ import annotations

import ctypes
import os
import re
from typing import Optional, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libposeidon.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "poseidon.h")

OK = 0
ERR_INVALID_ARG, ERR_NOT_INITIALIZED, ERR_CUDA, ERR_NCCL = -1, -2, -3, -4
ERR_SHAPE, ERR_ALIGNMENT, ERR_UNSUPPORTED, ERR_STATE = -5, -6, -7, -8
SCHEME_PS, SCHEME_SFB, SCHEME_SFPS = 0, 1, 2
LAYER_CONV, LAYER_FC = 0, 1
RECON_TF32, RECON_FP32 = 0, 1
FLAG_DWBP_OFF, FLAG_NO_PRIORITY, FLAG_NVLS_PS, FLAG_SYMM_SFB, FLAG_NVLS_SFB, FLAG_SSP1 = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
FLAG_SFPS, FLAG_EARLY_V, FLAG_INPLACE_FACTORS, FLAG_INPLACE_MN = 0x40, 0x80, 0x100, 0x200
STREAM_COMM, STREAM_RECON = 0, 1
SFB_PATH_NCCL, SFB_PATH_NCCL_SYMM, SFB_PATH_NVLS, SFB_PATH_SFPS = 0, 1, 2, 3
PS_ZERO_GRAD = 0x1

_STATUS_NAMES = {0: "OK", -1: "INVALID_ARG", -2: "NOT_INITIALIZED", -3: "CUDA", -4: "NCCL",
                 -5: "SHAPE", -6: "ALIGNMENT", -7: "UNSUPPORTED", -8: "STATE"}


class PoseidonError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"poseidon error {code} ({_STATUS_NAMES.get(code, '?')}): {msg}")
        self.code = code


class Costs(ctypes.Structure):
    _fields_ = [("sfb", ctypes.c_uint64), ("sf_ps", ctypes.c_uint64), ("full_ps", ctypes.c_uint64)]


class Hardware(ctypes.Structure):
    _fields_ = [("nvlink_gbps", ctypes.c_double), ("hbm_gbps", ctypes.c_double),
                ("tensor_tflops", ctypes.c_double), ("collective_latency_us", ctypes.c_double)]


class Topology(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nccl_id", ctypes.c_uint8 * 128), ("flags", ctypes.c_uint32)]


class IterStats(ctypes.Structure):
    _fields_ = [("exposed_ms", ctypes.c_float), ("sync_total_ms", ctypes.c_float),
                ("queue_ms", ctypes.c_float), ("recon_ms", ctypes.c_float),
                ("ps_update_ms", ctypes.c_float), ("first_ready_to_bwd_end_ms", ctypes.c_float),
                ("nccl_bytes_sent", ctypes.c_uint64), ("nccl_bytes_recv", ctypes.c_uint64),
                ("n_layers", ctypes.c_int32), ("iteration", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class LayerStats(ctypes.Structure):
    _fields_ = [("ready_to_start_ms", ctypes.c_float), ("comm_ms", ctypes.c_float),
                ("kernel_ms", ctypes.c_float), ("start_to_done_ms", ctypes.c_float),
                ("done_after_bwd_end_ms", ctypes.c_float), ("scheme", ctypes.c_int32),
                ("launched", ctypes.c_int32), ("pack_ms", ctypes.c_float)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1512_06216_b200/build.py` "
            "(there is no CPU fallback)")
    return ctypes.CDLL(LIB_PATH)


lib = _load()

_vp, _i32, _i64, _u32, _f, _u64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                   ctypes.c_float, ctypes.c_uint64)
_P = ctypes.POINTER
_SIGS = {
    "poseidon_init": (_i32, [_i32, _P(Topology), _P(_vp)]),
    "poseidon_choose_scheme": (_i32, [_i32, _i64, _i64, _i64, _i32, _P(Costs)]),
    "poseidon_choose_scheme_model": (_i32, [_i32, _i64, _i64, _i64, _i32, _P(Hardware),
                                            _P(ctypes.c_double), _P(ctypes.c_double)]),
    "poseidon_choose_scheme_model3": (_i32, [_i32, _i64, _i64, _i64, _i32, _P(Hardware), _P(ctypes.c_double),
                                             _P(ctypes.c_double), _P(ctypes.c_double)]),
    "poseidon_sync_fc_sfb": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _f, _vp]),
    "poseidon_sfb_post_input": (_i32, [_vp, _i32, _vp, _i64, _vp]),
    "poseidon_sync_ps": (_i32, [_vp, _i32, _vp, _vp, _i64, _f, _vp]),
    "poseidon_backprop_hook": (_i32, [_vp, _i32, _vp]),
    "poseidon_get_unique_id": (_i32, [_P(ctypes.c_uint8)]),
    "poseidon_shard_range": (_i32, [_i64, _i32, _i32, _P(_i64), _P(_i64), _P(_i64)]),
    "poseidon_register_layer": (_i32, [_vp, _i32, _i32, _i64, _i64, _i64, _i32, _i32, _P(_i32)]),
    "poseidon_sfb_slot": (_i32, [_vp, _i32, _P(_vp), _P(_i64), _P(_vp), _P(_i64)]),
    "poseidon_bind_ps_buffers": (_i32, [_vp, _i32, _vp, _vp, _i64, _u32]),
    "poseidon_bind_sfb_params": (_i32, [_vp, _i32, _vp, _vp]),
    "poseidon_set_lr": (_i32, [_vp, _f]),
    "poseidon_set_momentum": (_i32, [_vp, _i32, _f, _f]),
    "poseidon_ps_arena": (_i32, [_vp, _P(_i32)]),
    "poseidon_ps_layer_buffers": (_i32, [_vp, _i32, _P(_vp), _P(_vp), _P(_i64)]),
    "poseidon_nvls_status": (ctypes.c_char_p, [_vp]),
    "poseidon_sfb_path": (_i32, [_vp, _i32]),
    "poseidon_flush": (_i32, [_vp, _vp]),
    "poseidon_set_ps_buckets": (_i32, [_vp, _i64]),
    "poseidon_set_recon": (_i32, [_vp, _i32, _i32]),
    "poseidon_wait_layer": (_i32, [_vp, _i32, _vp]),
    "poseidon_iteration_end": (_i32, [_vp, _vp, _P(IterStats)]),
    "poseidon_get_iter_stats": (_i32, [_vp, _i32, _P(IterStats)]),
    "poseidon_get_layer_stats": (_i32, [_vp, _i32, _i32, _P(LayerStats)]),
    "poseidon_launch_count": (_u64, []),
    "poseidon_finalize": (_i32, [_vp]),
    "poseidon_last_error": (ctypes.c_char_p, []),
    "poseidon_version": (_i32, []),
    "poseidon_sfb_simulated": (_i32, [_vp, _vp, _i32, _i64, _i64, _i64, _vp, _vp, _f, _i32, _vp]),
    "poseidon_ps_simulated": (_i32, [_vp, _i32, _vp, _i64, _f, _vp]),
    "poseidon_ps_shard_update": (_i32, [_vp, _vp, _i64, _f, _vp, _vp]),
    "poseidon_reconstruct_sgd": (_i32, [_vp, _vp, _i32, _i64, _i64, _i64, _i64, _vp, _f, _i32, _vp]),
    "poseidon_pack_factors": (_i32, [_vp, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp]),
    "poseidon_reconstruct_sgd_rows": (_i32, [_vp, _vp, _i32, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _f, _i32,
                                             _vp]),
    "poseidon_stream": (_vp, [_vp, _i32]),
    "poseidon_set_staleness": (_i32, [_vp, _i32]),
    "poseidon_reconstruct_sgd_mn": (_i32, [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i64, _i64, _i64, _vp, _f,
                                           _vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def header_functions():
    """Names of every function include/poseidon.h declares."""
    with open(HEADER_PATH) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(poseidon_[a-z_0-9]+)\s*\(", text)))


def last_error() -> str:
    m = lib.poseidon_last_error()
    return m.decode() if m else ""


def _check(code: int):
    if code != OK:
        raise PoseidonError(code, last_error())
    return code


def _ptr(t) -> Optional[int]:
    """Device pointer of a tensor (None -> NULL); ints pass through.  The C ABI takes plain row-major fp32
    pointers, so a tensor must be float32 and contiguous (a strided view would be read as if it were not)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if getattr(t, "dtype", None) is not None and str(t.dtype) != "torch.float32":
        raise TypeError(f"libposeidon takes float32 buffers, got {t.dtype}")
    if hasattr(t, "is_contiguous") and not t.is_contiguous():
        raise ValueError("libposeidon takes contiguous row-major buffers (call .contiguous())")
    return t.data_ptr()


def _stream(s) -> Optional[int]:
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ------------------------------------------------------------ pure host ----
def choose_scheme(kind: int, M: int, N: int, K: int, P: int) -> Tuple[int, Tuple[int, int, int]]:
    c = Costs()
    r = lib.poseidon_choose_scheme(kind, M, N, K, P, ctypes.byref(c))
    if r < 0:
        raise PoseidonError(r, last_error())
    return r, (c.sfb, c.sf_ps, c.full_ps)


B200_HW = dict(nvlink_gbps=770.0, hbm_gbps=6543.7, tensor_tflops=669.6, collective_latency_us=10.0)


def choose_scheme_model(kind: int, M: int, N: int, K: int, P: int, hw: Optional[dict] = None):
    """Measured-cost model pick (scheme, t_sfb_us, t_ps_us); reported beside the paper's rule."""
    h = Hardware(**(hw or B200_HW))
    ts, tp = ctypes.c_double(), ctypes.c_double()
    r = lib.poseidon_choose_scheme_model(kind, M, N, K, P, ctypes.byref(h), ctypes.byref(ts), ctypes.byref(tp))
    if r < 0:
        raise PoseidonError(r, last_error())
    return r, ts.value, tp.value


def choose_scheme_model3(kind: int, M: int, N: int, K: int, P: int, hw: Optional[dict] = None):
    """Model pick among PS / SFB / SF-PS: (scheme, t_sfb_us, t_ps_us, t_sfps_us); reported beside the rule."""
    h = Hardware(**(hw or B200_HW))
    ts, tp, tf = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    r = lib.poseidon_choose_scheme_model3(kind, M, N, K, P, ctypes.byref(h), ctypes.byref(ts), ctypes.byref(tp),
                                          ctypes.byref(tf))
    if r < 0:
        raise PoseidonError(r, last_error())
    return r, ts.value, tp.value, tf.value


def shard_range(n: int, P: int, rank: int) -> Tuple[int, int, int]:
    b, e, p = _i64(), _i64(), _i64()
    _check(lib.poseidon_shard_range(n, P, rank, ctypes.byref(b), ctypes.byref(e), ctypes.byref(p)))
    return b.value, e.value, p.value


def get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib.poseidon_get_unique_id(buf))
    return bytes(buf)


def launch_count() -> int:
    return int(lib.poseidon_launch_count())


# ------------------------------------------------------------- context ----
class Context:
    """One libposeidon context (one process / GPU)."""

    def __init__(self, rank: int = 0, world: int = 1, device: int = 0, nccl_id: Optional[bytes] = None,
                 flags: int = 0):
        topo = Topology()
        topo.rank, topo.world, topo.device, topo.flags = rank, world, device, flags
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes")
            ctypes.memmove(topo.nccl_id, nccl_id, 128)
        h = _vp()
        _check(lib.poseidon_init(world, ctypes.byref(topo), ctypes.byref(h)))
        self.h = h
        self.rank, self.world, self.device, self.flags = rank, world, device, flags
        self._shapes = {}

    def close(self):
        if getattr(self, "h", None):
            lib.poseidon_finalize(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def register_layer(self, layer_id, kind, M, N, K, has_bias=True, scheme_override=-1) -> int:
        out = _i32()
        _check(lib.poseidon_register_layer(self.h, layer_id, kind, M, N, K, int(bool(has_bias)),
                                           scheme_override, ctypes.byref(out)))
        self._shapes[layer_id] = (M, N, K)
        return out.value

    def _check_factor(self, layer_id, name, t, cols):
        """The C ABI reads a factor tensor as K rows x `cols` with the registered K: refuse any other shape
        (a short last batch would make the pack read past the end, a longer one would drop samples)."""
        if t is None or isinstance(t, int) or layer_id not in self._shapes:
            return
        K = self._shapes[layer_id][2]
        if tuple(t.shape) != (K, cols):
            raise ValueError(f"layer {layer_id}: {name} must be ({K}, {cols}) = (registered K, "
                             f"{'M' if name == 'U' else 'N'}), got {tuple(t.shape)}")

    def sfb_slot(self, layer_id):
        u, v, lu, lv = _vp(), _vp(), _i64(), _i64()
        _check(lib.poseidon_sfb_slot(self.h, layer_id, ctypes.byref(u), ctypes.byref(lu), ctypes.byref(v),
                                     ctypes.byref(lv)))
        return u.value, lu.value, v.value, lv.value

    def bind_ps_buffers(self, layer_id, grad, W, n, flags=0):
        _check(lib.poseidon_bind_ps_buffers(self.h, layer_id, _ptr(grad), _ptr(W), n, flags))

    def bind_sfb_params(self, layer_id, W, bias=None):
        _check(lib.poseidon_bind_sfb_params(self.h, layer_id, _ptr(W), _ptr(bias)))

    def ps_arena(self) -> bool:
        """Collective: allocate the PS arena; True if the fused NVLS path is active."""
        act = _i32()
        _check(lib.poseidon_ps_arena(self.h, ctypes.byref(act)))
        return bool(act.value)

    def ps_layer_buffers(self, layer_id):
        g, w, n = _vp(), _vp(), _i64()
        _check(lib.poseidon_ps_layer_buffers(self.h, layer_id, ctypes.byref(g), ctypes.byref(w), ctypes.byref(n)))
        return g.value, w.value, n.value

    def set_ps_buckets(self, bucket_bytes: int):
        """Sync runs of small PS layers as one flat buffer (call before ps_arena, same on every rank)."""
        _check(lib.poseidon_set_ps_buckets(self.h, int(bucket_bytes)))

    def set_staleness(self, s: int):
        """SSP staleness s (context created with FLAG_SSP1; before registering layers and before ps_arena)."""
        _check(lib.poseidon_set_staleness(self.h, int(s)))

    def flush(self, stream=None):
        """SSP: apply every layer's deferred update (collective; no-op without FLAG_SSP1)."""
        _check(lib.poseidon_flush(self.h, _stream(stream)))

    def stream(self, which=STREAM_RECON):
        """The library's comm / reconstruction stream as a torch.cuda.ExternalStream (e.g. for record_stream)."""
        import torch
        h = lib.poseidon_stream(self.h, which)
        if not h:
            raise PoseidonError(ERR_INVALID_ARG, "poseidon_stream: bad context or stream id")
        return torch.cuda.ExternalStream(h, device=torch.device("cuda", self.device))

    def sfb_path(self, layer_id) -> int:
        r = lib.poseidon_sfb_path(self.h, layer_id)
        _check(min(r, 0))
        return r

    def nvls_status(self) -> str:
        m = lib.poseidon_nvls_status(self.h)
        return m.decode() if m else ""

    def set_momentum(self, mu, weight_decay=0.0, layer_id=-1):
        _check(lib.poseidon_set_momentum(self.h, layer_id, float(mu), float(weight_decay)))

    def set_lr(self, lr):
        _check(lib.poseidon_set_lr(self.h, float(lr)))

    def set_recon(self, recon, layer_id=-1):
        _check(lib.poseidon_set_recon(self.h, layer_id, recon))

    def sync_fc_sfb(self, layer_id, U, V, W=None, bias=None, lr=0.0, producer=None):
        if layer_id in self._shapes:
            M, N, _ = self._shapes[layer_id]
            self._check_factor(layer_id, "U", U, M)
            self._check_factor(layer_id, "V", V, N)
        _check(lib.poseidon_sync_fc_sfb(self.h, layer_id, _ptr(U), _ptr(V), _ptr(W), _ptr(bias), float(lr),
                                        _stream(producer)))

    def sfb_post_input(self, layer_id, V, stream=None):
        """FLAG_EARLY_V: pack and broadcast the layer input V (K x N, row-major) now (forward time)."""
        if layer_id in self._shapes:
            self._check_factor(layer_id, "V", V, self._shapes[layer_id][1])
        _check(lib.poseidon_sfb_post_input(self.h, layer_id, _ptr(V), V.stride(0), _stream(stream)))

    def sync_ps(self, layer_id, grad, W, n, lr, producer=None):
        _check(lib.poseidon_sync_ps(self.h, layer_id, _ptr(grad), _ptr(W), n, float(lr), _stream(producer)))

    def backprop_hook(self, layer_id, stream=None):
        _check(lib.poseidon_backprop_hook(self.h, layer_id, _stream(stream)))

    def wait_layer(self, layer_id, consumer=None):
        _check(lib.poseidon_wait_layer(self.h, layer_id, _stream(consumer)))

    def iteration_end(self, compute=None, stats=False):
        out = IterStats() if stats else None
        _check(lib.poseidon_iteration_end(self.h, _stream(compute), ctypes.byref(out) if stats else None))
        return out.as_dict() if stats else None

    def iter_stats(self, ago=0):
        out = IterStats()
        _check(lib.poseidon_get_iter_stats(self.h, ago, ctypes.byref(out)))
        return out.as_dict()

    def layer_stats(self, layer_id, ago=0):
        out = LayerStats()
        _check(lib.poseidon_get_layer_stats(self.h, ago, layer_id, ctypes.byref(out)))
        return out.as_dict()


# ------------------------------------------------ kernel-level entries ----
def sfb_simulated(U_all, V_all, P, K, M, N, W, bias, lr, recon=RECON_TF32, stream=None):
    _check(lib.poseidon_sfb_simulated(_ptr(U_all), _ptr(V_all), P, K, M, N, _ptr(W), _ptr(bias), float(lr),
                                      recon, _stream(stream)))


def ps_simulated(grads, P, W, n, lr, stream=None):
    _check(lib.poseidon_ps_simulated(_ptr(grads), P, _ptr(W), n, float(lr), _stream(stream)))


def ps_shard_update(g, W, count, alpha, stats=None, stream=None):
    _check(lib.poseidon_ps_shard_update(_ptr(g), _ptr(W), count, float(alpha), _ptr(stats), _stream(stream)))


def reconstruct_sgd(Ug, Vg, P, K, ldk, M, N, W, alpha, recon=RECON_TF32, stream=None):
    _check(lib.poseidon_reconstruct_sgd(_ptr(Ug), _ptr(Vg), P, K, ldk, M, N, _ptr(W), float(alpha), recon,
                                        _stream(stream)))


def reconstruct_sgd_mn(U, V, P, K, M, N, W, alpha, stream=None):
    """K1 on MN-major factors: U [P, K, ldu] (or [K, ldu] at P = 1), V [P, K, ldv]; ld = the last stride."""
    ldu, ldv = U.stride(-2), V.stride(-2)
    ublk = U.stride(0) if U.dim() == 3 else K * ldu
    vblk = V.stride(0) if V.dim() == 3 else K * ldv
    _check(lib.poseidon_reconstruct_sgd_mn(_ptr(U), ldu, ublk, _ptr(V), ldv, vblk, P, K, M, N, _ptr(W),
                                           float(alpha), _stream(stream)))


def reconstruct_sgd_rows(Ug, Vg, P, K, ldk, M, m0, m1, N, W, alpha, recon=RECON_TF32, stream=None):
    _check(lib.poseidon_reconstruct_sgd_rows(_ptr(Ug), _ptr(Vg), P, K, ldk, M, m0, m1, N, _ptr(W), float(alpha),
                                             recon, _stream(stream)))


def pack_factors(U, V, K, ldk, u_dst, v_dst=None, colsum=None, round_tf32=True, stream=None):
    """K3 alone: U (K x M) -> u_dst (M x ldk), V (K x N) -> v_dst (N x ldk), optional column sums of U."""
    M = U.shape[1]
    N = V.shape[1] if V is not None else 0
    _check(lib.poseidon_pack_factors(_ptr(U), U.stride(0), M, _ptr(V), V.stride(0) if V is not None else 0, N, K,
                                     ldk, int(bool(round_tf32)), _ptr(u_dst), _ptr(v_dst), _ptr(colsum),
                                     _stream(stream)))


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper so torch can view library-owned memory."""

    def __init__(self, ptr: int, shape, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, shape):
    """A torch tensor aliasing library-owned device memory (e.g. an SFB slot)."""
    import torch
    return torch.as_tensor(_CudaArray(ptr, shape), device="cuda")
