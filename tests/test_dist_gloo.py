"""Row-sharded (N > 1) solve, world size 2 over gloo on CPU.

The CUDA kernels are replaced by the CPU test double (tests/_cpu_kernels.py)
so that what is tested is the host logic of the multi-GPU path: the row
partition, the packed all-reduce of the A^T outputs and row sums, the HVP
partial all-reduce inside CG, the sketch all-reduce.  The sharded trajectory
must equal the unsharded one (same iteration counts, iterates to roundoff)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(kind):
    sys.path.insert(0, os.path.join(HERE, "golden"))
    import cases

    name = {"lasso": "lasso_small", "logistic": "logistic_small", "enet": "enet_small"}[kind]
    spec = cases.SOLVE_CASES[name][0]()
    return spec, cases.options_for(name)


def _solve(spec, opts, shard=None):
    sys.path.insert(0, HERE)
    import paper_2310_08333_b200 as nys
    from _cpu_kernels import CpuKernels

    prob = nys.MLProblem(nys.builtin_loss(spec["loss"]), spec["A"], spec["b"], spec["lambda1"], spec["lambda2"])
    return nys.solve(prob, nys.SolverOptions(**opts), kernels=CpuKernels(), shard=shard)


def _worker(rank, world, port, kind, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_08333_b200.dist import current_shard

        spec, opts = _problem(kind)
        shard = current_shard(spec["A"].shape[0])
        assert shard.world == world and shard.sharded
        res = _solve(spec, opts, shard)
        if rank == 0:
            np.savez(out_path, x=res.x, z=res.z, it=res.iterations, obj=res.objective,
                     cg=np.array([h.cg_iters for h in res.history]), rows=shard.row_stop - shard.row_start)
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("kind", ["lasso", "logistic", "enet"])
def test_row_sharded_solve_matches_single(tmp_path, kind):
    torch.set_num_threads(1)
    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(2, _free_port(), kind, out), nprocs=2, join=True)
    got = np.load(out)
    spec, opts = _problem(kind)
    ref = _solve(spec, opts)
    assert int(got["rows"]) == (spec["A"].shape[0] + 1) // 2
    assert int(got["it"]) == ref.iterations
    np.testing.assert_array_equal(got["cg"], [h.cg_iters for h in ref.history])
    np.testing.assert_allclose(got["x"], ref.x, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(got["z"], ref.z, rtol=1e-9, atol=1e-12)
    assert abs(float(got["obj"]) - ref.objective) <= 1e-10 * abs(ref.objective)


def test_cpu_double_matches_oracle():
    """The CPU double drives the engine to the oracle's trajectory, so the
    gloo test above checks the real control flow."""
    from oracle import port

    spec, opts = _problem("logistic")
    res = _solve(spec, opts)
    o = port.solve(port.MLSpec(spec["loss"], spec["A"], spec["b"], spec["lambda1"], spec["lambda2"]),
                   port.Options(**opts))
    assert res.iterations == o.iterations
    assert abs(res.objective - o.objective) <= 1e-9 * abs(o.objective)


def test_row_range_partition():
    from paper_2310_08333_b200.dist import row_range

    for N in (1, 7, 100, 12500 * 8):
        for world in (1, 2, 3, 4, 8):
            spans = [row_range(N, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
