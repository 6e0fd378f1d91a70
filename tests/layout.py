"""Test helpers: decode the library's device layouts (include/sage3.h) into the oracle's logical layouts.
Pure index manipulation — no arithmetic of the method."""
import numpy as np


def unpack_codes(packed: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """[rows][cols/2] bytes, element 2k in the low nibble -> [rows][cols] codes."""
    p = np.asarray(packed, np.uint8).reshape(rows, cols // 2)
    out = np.empty((rows, cols), np.uint8)
    out[:, 0::2] = p & 0xF
    out[:, 1::2] = p >> 4
    return out


def sf_atoms_to_logical(raw: np.ndarray, R: int, C: int) -> np.ndarray:
    """SF-atom bytes of one R x C scale matrix (R % 128 == 0, C % 4 == 0) -> logical [R][C]."""
    raw = np.asarray(raw, np.uint8).reshape(-1)
    r = np.arange(R)[:, None]
    c = np.arange(C)[None, :]
    off = ((r // 128) * (C // 4) + c // 4) * 512 + (r % 32) * 16 + ((r // 32) % 4) * 4 + (c % 4)
    return raw[off]


def decode_head(qkv, bh: int):
    """Logical codes/scales of head bh from an FP4QKV (torch buffers) -> dict of numpy arrays."""
    Np, d = qkv.N_pad, qkv.d
    qd = qkv.q_data.view(-1, Np, d // 2)[bh].cpu().numpy()
    kd = qkv.k_data.view(-1, Np, d // 2)[bh].cpu().numpy()
    vd = qkv.v_data.view(-1, d, Np // 2)[bh].cpu().numpy()
    qs = qkv.q_sf.view(-1, Np * d // 16)[bh].cpu().numpy()
    ks = qkv.k_sf.view(-1, Np * d // 16)[bh].cpu().numpy()
    vs = qkv.v_sf.view(-1, 128 * Np // 16)[bh].cpu().numpy()
    km = qkv.k_mean.view(torch_float32()).view(-1, d)[bh].cpu().numpy()
    out = {
        "q_codes": unpack_codes(qd, Np, d), "k_codes": unpack_codes(kd, Np, d), "v_codes": unpack_codes(vd, d, Np),
        "q_sf": sf_atoms_to_logical(qs, Np, d // 16), "k_sf": sf_atoms_to_logical(ks, Np, d // 16),
        "v_sf_full": sf_atoms_to_logical(vs, 128, Np // 16), "km": km,
    }
    if getattr(qkv, "smooth_q", False):  # smoothing Q: q̄ per tile and the GEMV term
        T = Np // 128
        out["q_mean"] = qkv.q_mean.view(torch_float32()).view(-1, T, d)[bh].cpu().numpy()
        out["ds"] = qkv.ds.view(torch_float32()).view(-1, T, Np)[bh].cpu().numpy()
    return out


def torch_float32():
    import torch

    return torch.float32
