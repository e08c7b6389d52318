"""Parity gates shared by the GPU tests (reading Z13 / Z13b).

check_update() applies the max-normalised update metric AND refuses a case whose fp32 ulp excuse
(oracle.ulp_excuse) exceeds 0.1 x the gate: such a case would not test the gate it states
(W ~ N(0,1) with dW ~ 1e-4 made the 1e-5 gate ~100x looser).  w0_like() scales a random
starting W to a few times the update, so random fp32 cases stay tight while W still enters the result.
"""
import numpy as np

import oracle as O

TOL_FP32 = 1e-5
TOL_TF32 = 2e-3


def check_update(W0, out, ref, tol, what=""):
    excuse = O.ulp_excuse(W0, ref)
    assert excuse <= 0.1 * tol, (f"{what}: mis-parameterised parity case, the fp32 ulp excuse is {excuse:.2e} "
                                 f"of max|dW| (> 0.1 x gate {tol:g}): make |W'| closer to |dW|")
    err = O.update_error_fp32(W0, out, ref)
    assert err <= tol, f"{what}: update error {err:.3e} > {tol:g}"
    return err


def w0_like(W, dW, factor=4.0):
    """W rescaled so that max|W| = factor * max|dW| (float32); dW = the reference update."""
    W = np.asarray(W, np.float64)
    m = float(np.max(np.abs(W))) or 1.0
    d = float(np.max(np.abs(np.asarray(dW, np.float64)))) or 1.0
    return (W * (factor * d / m)).astype(np.float32)
