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
