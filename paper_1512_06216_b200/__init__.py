"""paper_1512_06216_b200 — B200-native Poseidon gradient synchronisation.

The product is ``libposeidon.so`` (C ABI, ``include/poseidon.h``); this package
holds its CUDA/C++ sources (``csrc/``), the ctypes binding (``binding``) and
the DWBP glue that drives it from PyTorch autograd (``dwbp``).
"""
from .binding import (  # noqa: F401
    LAYER_CONV, LAYER_FC, SCHEME_PS, SCHEME_SFB, SCHEME_SFPS, RECON_TF32, RECON_FP32, FLAG_DWBP_OFF,
    FLAG_NO_PRIORITY, FLAG_NVLS_PS, FLAG_SYMM_SFB, FLAG_NVLS_SFB, FLAG_SSP1, FLAG_SFPS, FLAG_EARLY_V, FLAG_INPLACE_FACTORS, FLAG_INPLACE_MN, SFB_PATH_NCCL,
    SFB_PATH_NCCL_SYMM, SFB_PATH_NVLS, SFB_PATH_SFPS, PS_ZERO_GRAD, Context, PoseidonError, choose_scheme,
    shard_range, get_unique_id, launch_count, sfb_simulated, ps_simulated, ps_shard_update, reconstruct_sgd,
    reconstruct_sgd_rows, reconstruct_sgd_mn, pack_factors, STREAM_COMM, STREAM_RECON,
)
