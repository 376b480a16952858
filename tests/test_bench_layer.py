"""Benchmark harness (generators, file ingestion, records, runner, CLI) against
the reference's own outputs (tests/golden/bench_runs.npz, written by
make_golden.py from nysopt.bench).  The host-side pieces run on CPU; the
runner and CLI solve on the B200 (gpu marker)."""

import json
import os

import numpy as np
import pytest

from conftest import load_golden

from paper_2310_08333_b200.bench import (CSV_HEADER, BenchConfig, RunRecord, gen_bounded_ls, gen_huber_data,
                                         gen_logistic_data, gen_portfolio_data, gen_regression_data, read_libsvm,
                                         read_qp_files, write_libsvm)
from paper_2310_08333_b200.errors import DataError, InputError


def test_generators_match_reference():
    g = load_golden("bench_runs.npz")
    A, b = gen_regression_data(20, 10, 1)
    np.testing.assert_array_equal(A, g["reg_A"])
    np.testing.assert_array_equal(b, g["reg_b"])
    A, b, lam = gen_huber_data(20, 3)
    np.testing.assert_array_equal(A, g["hub_A"])
    np.testing.assert_array_equal(b, g["hub_b"])
    assert lam == float(g["hub_lam"])
    d, F, mu, gamma = gen_portfolio_data(1, 2)
    np.testing.assert_array_equal(d, g["pf_d"])
    np.testing.assert_array_equal(F, g["pf_F"])
    np.testing.assert_array_equal(mu, g["pf_mu"])
    assert gamma == 1.0
    A, lam = gen_logistic_data(20, 10, 4)
    np.testing.assert_array_equal(A, g["log_A"])
    assert lam == float(g["log_lam"])
    qp = gen_bounded_ls(20, 5)
    np.testing.assert_array_equal(qp.P.a, g["bls_P"])
    np.testing.assert_array_equal(qp.q, g["bls_q"])
    with pytest.raises(DataError):
        gen_huber_data(7, 0)
    with pytest.raises(DataError):
        gen_portfolio_data(0, 0)


def test_libsvm_single_entry_and_label_only(tmp_path):
    p = tmp_path / "a.svm"
    p.write_text("1.5 3:2.0\n-1\n")
    op, y = read_libsvm(p)
    assert op.a.shape == (2, 3)
    np.testing.assert_array_equal(op.a.toarray(), [[0, 0, 2.0], [0, 0, 0]])
    np.testing.assert_array_equal(y, [1.5, -1.0])


@pytest.mark.parametrize("text,where", [("1 0:1.0\n", ":1:"), ("x 1:1\n", ":1:"), ("1 1:1\n1 2-3\n", ":2:")])
def test_libsvm_malformed_reports_line(tmp_path, text, where):
    p = tmp_path / "bad.svm"
    p.write_text(text)
    with pytest.raises(InputError, match=where):
        read_libsvm(p)


def test_libsvm_roundtrip_exact(tmp_path):
    import scipy.sparse as sp

    rng = np.random.default_rng(0)
    A = sp.random(30, 12, density=0.3, random_state=1, format="csr")
    A.data = rng.standard_normal(A.nnz)
    b = rng.standard_normal(30)
    p = tmp_path / "rt.svm"
    write_libsvm(p, A, b)
    op, y = read_libsvm(p, n_features=12)
    np.testing.assert_array_equal(op.a.toarray(), A.toarray())
    np.testing.assert_array_equal(y, b)
    with pytest.raises(InputError):
        read_libsvm(p, n_features=3)


def _write_qp(tmp_path, P, q, M, l, u):
    import scipy.io
    import scipy.sparse as sp

    scipy.io.mmwrite(str(tmp_path / "P.mtx"), sp.csr_matrix(P))
    scipy.io.mmwrite(str(tmp_path / "M.mtx"), sp.csr_matrix(M))
    for name, v in (("q", q), ("l", l), ("u", u)):
        (tmp_path / f"{name}.txt").write_text("\n".join(repr(float(x)) for x in v) + "\n")


def test_qp_files(tmp_path):
    _write_qp(tmp_path, np.eye(2), [1.0, -1.0], np.eye(2), [-np.inf, 0.0], [1.0, np.inf])
    qp = read_qp_files(*(tmp_path / f for f in ("P.mtx", "q.txt", "M.mtx", "l.txt", "u.txt")))
    assert qp.n == 2 and qp.m == 2
    assert np.isinf(qp.box.l[0]) and np.isinf(qp.box.u[1])
    (tmp_path / "q.txt").write_text("1\n2\n3\n")
    with pytest.raises(InputError):
        read_qp_files(*(tmp_path / f for f in ("P.mtx", "q.txt", "M.mtx", "l.txt", "u.txt")))
    _write_qp(tmp_path, [[1.0, 0.5], [0.0, 1.0]], [0.0, 0.0], np.eye(2), [0, 0], [1, 1])
    with pytest.warns(UserWarning):
        qp = read_qp_files(*(tmp_path / f for f in ("P.mtx", "q.txt", "M.mtx", "l.txt", "u.txt")))
    np.testing.assert_allclose(qp.P.a.toarray(), [[1.0, 0.25], [0.25, 1.0]])


def test_csv_header_and_record_roundtrip(tmp_path):
    assert CSV_HEADER.split(",") == ["problem", "n", "status", "iters", "setup_s", "precond_s", "linsys_total_s",
                                     "linsys_avg_ms", "prox_total_s", "prox_avg_ms", "total_s", "rp", "rd",
                                     "objective"]
    rec = RunRecord("lasso", 10, "optimal", 5, 0.1, 0.01, 0.2, 40.0, 0.001, 0.2, 0.5, 1e-5, 2e-5, 3.25,
                    seed=3, history=[{"k": 1}])
    assert RunRecord.from_json(rec.to_json()) == rec
    lines = rec.to_csv().splitlines()
    assert lines[0] == CSV_HEADER and len(lines[1].split(",")) == 14
    assert json.loads(rec.to_json())["history"] == [{"k": 1}]


def test_config_validation():
    for kw in (dict(problem="nope", n=3), dict(problem="lasso"), dict(problem="portfolio"),
               dict(problem="lasso", n=3, data="x"), dict(problem="lasso", n=-1), dict(problem="lasso", n=3, fmt="x"),
               dict(problem="portfolio", k=1, portfolio_path="x")):
        with pytest.raises(InputError):
            BenchConfig(**kw)
    BenchConfig(problem="portfolio", k=2)


RUNS = [("lasso", dict(n=60)), ("elastic_net", dict(n=50)), ("logistic", dict(n=40)), ("huber", dict(n=60)),
        ("bounded_ls", dict(n=80)), ("portfolio", dict(k=1, portfolio_path="qp")),
        ("portfolio", dict(k=1, portfolio_path="operators")), ("lasso", dict(n=40, norm="linf", tol=1e-6))]


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(RUNS)))
def test_run_bench_matches_reference(i, tmp_path):
    from paper_2310_08333_b200.bench import run_bench

    g = load_golden("bench_runs.npz")
    prob, kw = RUNS[i]
    out = tmp_path / "rec.csv"
    rec = run_bench(BenchConfig(problem=prob, seed=3, out=str(out), **kw))
    assert rec.status == str(g[f"run{i}_status"])
    assert rec.n == int(g[f"run{i}_n"])
    assert abs(rec.iters - int(g[f"run{i}_iters"])) <= 2, (rec.iters, int(g[f"run{i}_iters"]))
    ref = float(g[f"run{i}_objective"])
    assert abs(rec.objective - ref) <= 1e-6 * abs(ref)
    assert out.read_text().splitlines()[0] == CSV_HEADER
    assert rec.total_s >= rec.setup_s >= 0 and rec.linsys_total_s <= rec.total_s


@pytest.mark.gpu
def test_cli_exit_codes(tmp_path):
    from click.testing import CliRunner

    from paper_2310_08333_b200.cli import main

    r = CliRunner()
    res = r.invoke(main, ["bench", "lasso", "--n", "40", "--out", str(tmp_path / "o.json"), "--format", "json"])
    assert res.exit_code == 0, res.output
    assert res.output.splitlines()[0] == CSV_HEADER
    assert json.loads((tmp_path / "o.json").read_text())["status"] == "optimal"
    assert r.invoke(main, ["bench", "lasso", "--n", "40", "--max-iter", "2"]).exit_code == 3
    assert r.invoke(main, ["bench", "lasso"]).exit_code == 4
    assert r.invoke(main, ["bench", "lasso", "--n", "5", "--plot"]).exit_code == 4
    # infeasible QP from files: exit 2 (cli.py:17-24)
    _write_qp(tmp_path, np.zeros((1, 1)), [0.0], np.array([[1.0], [1.0]]), [-np.inf, 1.0], [-1.0, np.inf])
    res = r.invoke(main, ["bench", "qp_file", "--data", str(tmp_path), "--max-iter", "2000"])
    assert res.exit_code == 2, res.output
    # libsvm input
    import scipy.sparse as sp

    rng = np.random.default_rng(2)
    A = sp.random(40, 15, density=0.4, random_state=3, format="csr")
    write_libsvm(tmp_path / "d.svm", A, A @ rng.standard_normal(15))
    assert r.invoke(main, ["bench", "lasso", "--data", str(tmp_path / "d.svm")]).exit_code == 0
