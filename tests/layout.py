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
    """SF-atom bytes of one R x C scale matrix (R % 128 == 0; the atoms hold C4 = round_up(C, 4) columns)
    -> logical [R][C4] (columns >= C are the atom padding)."""
    raw = np.asarray(raw, np.uint8).reshape(-1)
    C4 = (C + 3) // 4 * 4
    r = np.arange(R)[:, None]
    c = np.arange(C4)[None, :]
    off = ((r // 128) * (C4 // 4) + c // 4) * 512 + (r % 32) * 16 + ((r // 32) % 4) * 4 + (c % 4)
    return raw[off]


def decode_head(qkv, bh: int):
    """Logical codes/scales of head bh from an FP4QKV (torch buffers) -> dict of numpy arrays."""
    Np, d = qkv.N_pad, qkv.d
    G = 32 if getattr(qkv, "fmt", 0) == 1 else 16  # MXFP4 / NVFP4 block size
    C = d // G
    qd = qkv.q_data.view(-1, Np, d // 2)[bh].cpu().numpy()
    kd = qkv.k_data.view(-1, Np, d // 2)[bh].cpu().numpy()
    vd = qkv.v_data.view(-1, d, Np // 2)[bh].cpu().numpy()
    BH = qkv.q_data.numel() // (Np * d // 2)
    qs = qkv.q_sf.view(BH, -1)[bh].cpu().numpy()
    ks = qkv.k_sf.view(BH, -1)[bh].cpu().numpy()
    vs = qkv.v_sf.view(BH, -1)[bh].cpu().numpy()
    km = qkv.k_mean.view(torch_float32()).view(-1, d)[bh].cpu().numpy()
    q_sf4, k_sf4 = sf_atoms_to_logical(qs, Np, C), sf_atoms_to_logical(ks, Np, C)
    out = {
        "q_codes": unpack_codes(qd, Np, d), "k_codes": unpack_codes(kd, Np, d), "v_codes": unpack_codes(vd, d, Np),
        "q_sf": q_sf4[:, :C], "k_sf": k_sf4[:, :C], "sf_pad": np.concatenate([q_sf4[:, C:], k_sf4[:, C:]], 1),
        "v_sf_full": sf_atoms_to_logical(vs, 128, Np // G), "km": km,
    }
    if getattr(qkv, "smooth_q", False):  # smoothing Q: q̄ per tile and the GEMV term
        T = Np // 128
        out["q_mean"] = qkv.q_mean.view(torch_float32()).view(-1, T, d)[bh].cpu().numpy()
        out["ds"] = qkv.ds.view(torch_float32()).view(-1, T, Np)[bh].cpu().numpy()
    return out


def torch_float32():
    import torch

    return torch.float32
