"""Back-projection (BPA) brute force -- the paper's gold standard (P:199-200,
P:380) used only to pin the oracle on tiny inputs.

TEST INFRASTRUCTURE ONLY -- never imported by the product path.

o_BPA(v) = sum_{t,r,p,i} s[t,r,p,i] * exp(+j k_i (|v - tx_w| + |v - rx_w|))

with the ACTUAL (jittered) Tx/Rx world positions and Eq. (2) distances
(P:113-121): the matched filter of Eq. (9).  The geometric
recurrence exp(+j k_i R) = exp(+j k_0 R) * exp(+j dk R)^i replaces one complex
exponential per frequency (exact up to rounding).
"""
from __future__ import annotations

import numpy as np


def bpa(s_frame: np.ndarray, tx_w: np.ndarray, rx_w: np.ndarray, k: np.ndarray,
        voxels: np.ndarray, voxel_chunk: int = 4096) -> np.ndarray:
    """s_frame: [n_tx, n_rx, P, n_k]; tx_w: [n_tx, P, 3]; rx_w: [n_rx, P, 3];
    voxels: [V, 3].  Returns complex128 [V]."""
    nt, nr, P, nk = s_frame.shape
    k0 = float(k[0])
    dk = (k[-1] - k[0]) / (nk - 1) if nk > 1 else 0.0
    out = np.zeros(voxels.shape[0], complex)
    for v0 in range(0, voxels.shape[0], voxel_chunk):
        vox = voxels[v0:v0 + voxel_chunk]
        for t in range(nt):
            dT = np.linalg.norm(vox[None, :, :] - tx_w[t][:, None, :], axis=-1)      # [P, V]
            for r in range(nr):
                R = dT + np.linalg.norm(vox[None, :, :] - rx_w[r][:, None, :], axis=-1)
                cur = np.exp(1j * k0 * R)
                step = np.exp(1j * dk * R)
                row = s_frame[t, r].astype(complex)                                   # [P, nk]
                acc = np.zeros(vox.shape[0], complex)
                for i in range(nk):
                    acc += row[:, i] @ cur
                    cur *= step
                out[v0:v0 + voxel_chunk] += acc
    return out
