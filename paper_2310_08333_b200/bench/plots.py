"""Convergence figures for a run record (``bench/plots.py``): residual and
objective traces written next to the tabular output."""

from __future__ import annotations

from .records import RunRecord


def render_run_plots(record: RunRecord, out_prefix: str) -> list:
    if not record.history:
        return []
    try:
        import matplotlib
    except ImportError:  # not in every image; the record itself is unaffected
        from ..errors import CapabilityError

        raise CapabilityError("--plot needs matplotlib, which is not installed") from None
    matplotlib.use("Agg")
    import matplotlib.pyplot as plt

    ks = [h["k"] for h in record.history]
    fig, (a, b) = plt.subplots(1, 2, figsize=(9, 3.5))
    a.semilogy(ks, [max(h["rp_norm"], 1e-300) for h in record.history], label="primal residual")
    a.semilogy(ks, [max(h["rd_norm"], 1e-300) for h in record.history], label="dual residual")
    a.set_xlabel("iteration")
    a.set_ylabel("residual norm")
    a.legend()
    b.plot(ks, [h["objective"] for h in record.history])
    b.set_xlabel("iteration")
    b.set_ylabel("objective")
    fig.suptitle(f"{record.problem} (n={record.n}, status={record.status})")
    fig.tight_layout()
    path = f"{out_prefix}_convergence.png"
    fig.savefig(path, dpi=130)
    plt.close(fig)
    return [path]
