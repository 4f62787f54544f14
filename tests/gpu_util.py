"""Helpers for GPU tests: move generated bf16 bit arrays into device / pinned memory."""
import numpy as np
import torch


def dev(bits) -> torch.Tensor:
    """uint16 bit array -> device int16 tensor holding the same bits (bf16 storage)."""
    a = np.ascontiguousarray(bits, dtype=np.uint16)
    return torch.from_numpy(a.view(np.int16)).to("cuda")


def dev_f32(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to("cuda")


def pinned(bits) -> torch.Tensor:
    a = np.ascontiguousarray(bits, dtype=np.uint16)
    t = torch.empty(a.shape, dtype=torch.int16, pin_memory=True)
    t.numpy()[...] = a.view(np.int16)
    return t


def bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint16)


def split_weight(W, n_res):
    """(W_dev rows [0,n_res) on device or None, W_host rows [n_res,N) pinned or None)."""
    N = W.shape[0]
    W_dev = dev(W[:n_res]) if n_res > 0 else None
    W_host = pinned(W[n_res:]) if n_res < N else None
    return W_dev, W_host
