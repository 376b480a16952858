"""Config 5 generated in HBM, bit-for-bit the host recipe of ``datagen.cfg5_block``.

Config 5 (BASELINE.json configs[4]) is a 100000 x 200000 FP64 matrix: 160 GB,
which one B200 (180 GB) can hold but no host can build and upload in a
reasonable time.  BASELINE.json says it is "generated per shard from the
seed": row block j (12500 rows) is ``default_rng([4, j]).standard_normal`` of
the block followed by the block's noise draws (``datagen.cfg5_block``).  This
module produces exactly those numbers on the GPU with the PCG64 + ziggurat
generator of ``csrc/rng.cu`` (``nys_gaussian_draws_f64``), in pieces that
chain exactly: each piece reports the 64-bit draws it consumed and the next
piece starts from the PCG64 state advanced by that many steps
(``numpy.random.PCG64.advance``).  A rank of a row-sharded run generates only
its own blocks.  Not on the solve's hot path: it builds the input.
"""

from __future__ import annotations

import numpy as np
import torch

from . import datagen

CFG5_N = 200000
CFG5_ROWS = 100000
CFG5_BLOCK_ROWS = CFG5_ROWS // datagen.CFG5_BLOCKS  # 12500
PIECE = 1 << 26  # samples per generator call (~1.1 GB of workspace)


def _state(bg: np.random.PCG64) -> tuple[int, int]:
    st = bg.state["state"]
    return int(st["state"]), int(st["inc"])


def normals_into(kx, bg: np.random.PCG64, out: torch.Tensor, piece: int = PIECE) -> None:
    """Fill the contiguous CUDA tensor ``out`` with the next ``out.numel()``
    standard normals of ``bg``'s stream and advance ``bg`` past them (so the
    host generator continues where the device left off)."""
    flat = out.view(-1)
    total = flat.numel()
    pos = 0
    while pos < total:
        cnt = min(piece, total - pos)
        s, inc = _state(bg)
        draws = kx.gaussian_stream(s, inc, flat[pos:pos + cnt])
        bg.advance(draws)
        pos += cnt


def cfg5_block_into(kx, j: int, out: torch.Tensor, rows_per_block: int = CFG5_BLOCK_ROWS,
                    n: int = CFG5_N, piece: int = PIECE) -> torch.Tensor:
    """Row block j of config 5 into ``out`` (rows_per_block x n, contiguous,
    CUDA); returns the block's noise (CUDA, rows_per_block).  Same values as
    ``datagen.cfg5_block(j, rows_per_block, n)``."""
    assert out.is_contiguous() and tuple(out.shape) == (rows_per_block, n)
    bg = np.random.PCG64([4, j])  # the bit generator of default_rng([4, j])
    normals_into(kx, bg, out, piece)
    out.mul_(1.0 / np.sqrt(100000))
    noise = torch.empty(rows_per_block, dtype=torch.float64, device=out.device)
    normals_into(kx, bg, noise, piece)
    noise.mul_(0.01)
    return noise


def cfg5_device(kx, blocks=None, rows_per_block: int = CFG5_BLOCK_ROWS, n: int = CFG5_N,
                piece: int = PIECE):
    """The rows of config 5 held by this process: blocks ``blocks`` (default:
    all 8) stacked in one (len(blocks) * rows_per_block) x n CUDA tensor, and
    b = A x_true + noise for those rows (on the device).  x_true is the host
    ``datagen.cfg5_truth`` vector."""
    blocks = list(range(datagen.CFG5_BLOCKS)) if blocks is None else list(blocks)
    dev = kx.device
    A = torch.empty(len(blocks) * rows_per_block, n, dtype=torch.float64, device=dev)
    noise = torch.empty(len(blocks) * rows_per_block, dtype=torch.float64, device=dev)
    for k, j in enumerate(blocks):
        sl = slice(k * rows_per_block, (k + 1) * rows_per_block)
        noise[sl] = cfg5_block_into(kx, j, A[sl], rows_per_block, n, piece)
    xt = torch.from_numpy(datagen.cfg5_truth(n)).to(dev)
    b = torch.empty(1, A.shape[0], dtype=torch.float64, device=dev)
    kx.gemv(A, xt.view(1, -1), b)
    b = b.view(-1) + noise
    return A, b, xt


def lasso_device(kx, N: int, n: int, seed: int, nnz_frac: float, rows=None, host_b: bool = False):
    """Configs 1 and 4 (``datagen.lasso_data``) with A generated in HBM: the
    first N*n draws of ``default_rng(seed)`` (scaled by 1/sqrt(N) exactly as
    the host recipe), then support, values and noise from the same host
    stream.  Returns (A rows [rows] on the device, b (host, N), lambda,
    x_true).  ``host_b``: b and lambda from a host copy of A with NumPy
    (bitwise the host recipe; needs the 8 N n bytes on the host, returned as
    the fifth value), else from the device GEMVs (roundoff-level
    differences).  Every rank of a sharded run computes the same b and lambda
    and keeps only its rows."""
    dev = kx.device
    bg = np.random.PCG64(seed)
    A = torch.empty(N, n, dtype=torch.float64, device=dev)
    normals_into(kx, bg, A)
    A.mul_(1.0 / np.sqrt(N))
    rng = np.random.Generator(bg)
    k = max(1, int(round(nnz_frac * n)))
    support = rng.choice(n, size=k, replace=False)
    x_true = np.zeros(n)
    x_true[support] = rng.standard_normal(k)
    noise = 0.01 * rng.standard_normal(N)
    A_host = None
    if host_b:
        A_host = torch.empty(N, n, dtype=torch.float64, pin_memory=True)
        A_host.copy_(A)
        Ah = A_host.numpy()
        b = Ah @ x_true + noise
        lam = 0.1 * float(np.max(np.abs(Ah.T @ b)))
    else:
        bt = torch.empty(1, N, dtype=torch.float64, device=dev)
        kx.gemv(A, torch.from_numpy(x_true).to(dev).view(1, -1), bt)
        b = bt.view(-1).cpu().numpy() + noise
        atb = torch.empty(1, n, dtype=torch.float64, device=dev)
        kx.gemvT(A, torch.from_numpy(b).to(dev).view(1, -1), atb)
        lam = 0.1 * float(atb.abs().max())
    if rows is not None and tuple(rows) != (0, N):
        A = A[rows[0]:rows[1]].clone()
        torch.cuda.empty_cache()
    return A, b, lam, x_true, A_host

