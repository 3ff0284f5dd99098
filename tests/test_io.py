"""Ingestion row: Matrix Market / CSV through the C ABI and the
`symsplit_b200` CLI, mirroring reference tests/unit/test_io.cpp:51-155 and the
CLI flag surface of tools/main.cpp:157-259 / acceptance.cpp:382-420 (criterion 9).

CSV and the CLI's usage/io exit paths are host-only and run here; everything
that creates a device matrix is marked gpu."""
import json
import os
import subprocess

import numpy as np
import pytest

import pyoracle as O
from helpers import oracle_workload

import paper_1902_10559_b200 as P
from paper_1902_10559_b200.configs import CONFIGS

CLI = os.path.join(os.path.dirname(P.__file__), "symsplit_b200")


def spit(path, text):
    with open(path, "w") as fh:
        fh.write(text)


def cli(*args, env=None):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600,
                          env=env)


def mm_bytes(rows, cols, ptr, idx, val):
    """Matrix Market text the reference writer produces (io.cpp:189-210) for a
    CSR matrix: non-zeros in (row, col) order, 1-based, %.17g."""
    lines = []
    for i in range(rows):
        for k in range(ptr[i], ptr[i + 1]):
            if val[k] != 0.0:
                lines.append("%d %d %.17g" % (i + 1, idx[k] + 1, val[k]))
    head = "%%%%MatrixMarket matrix coordinate real general\n%d %d %d\n" % (rows, cols, len(lines))
    return (head + "".join(x + "\n" for x in lines)).encode()


def config_text(w):
    return ("# %s\nk %d\ngamma_deg %.17g\nh_e %.17g\nh_m %.17g\nl_m %.17g\nn_p %d\n"
            "obj_size %.17g\ngrid_nx %d\ngrid_ny %d\n" % (
                w.name, w.k, w.gamma_deg, w.h_e, w.h_m, w.l_m, w.bins, w.obj_size, w.grid_nx,
                w.grid_ny))


# ------------------------------------------------------------------ CSV (host only)
def test_vector_csv_roundtrip(tmp_path):
    path = str(tmp_path / "p.csv")
    P.write_vector_csv([5, 6, 8, 7], path)
    assert np.array_equal(P.read_vector_csv(path), [5.0, 6.0, 8.0, 7.0])
    spit(tmp_path / "empty.csv", "")
    assert P.read_vector_csv(str(tmp_path / "empty.csv")).size == 0
    big = np.random.default_rng(5002).uniform(-1e12, 1e12, 100000)
    P.write_vector_csv(big, path)
    back = P.read_vector_csv(path)
    assert back.shape == big.shape and back.tobytes() == big.tobytes()
    spit(tmp_path / "crlf.csv", "1.5\r\n\r\n-2 \n")
    assert np.array_equal(P.read_vector_csv(str(tmp_path / "crlf.csv")), [1.5, -2.0])


def test_vector_csv_errors_carry_line_numbers(tmp_path):
    spit(tmp_path / "bad.csv", "1.5\nx\n")
    with pytest.raises(P.IoError, match="line 2: not a number: 'x'"):
        P.read_vector_csv(str(tmp_path / "bad.csv"))
    spit(tmp_path / "trail.csv", "1.5\n\n2.5abc\n")
    with pytest.raises(P.IoError, match="line 3: trailing content in '2.5abc'"):
        P.read_vector_csv(str(tmp_path / "trail.csv"))
    with pytest.raises(P.IoError, match="cannot open file for reading"):
        P.read_vector_csv(str(tmp_path / "missing.csv"))
    with pytest.raises(P.IoError, match="cannot open file for writing"):
        P.write_vector_csv([1.0], str(tmp_path / "no" / "such" / "dir.csv"))


# ------------------------------------------------------------------ CLI exit codes (host only)
def test_cli_usage_and_io_exit_codes(tmp_path):
    assert os.path.exists(CLI), "symsplit_b200 CLI not built (make -C paper_1902_10559_b200/csrc)"
    assert cli().returncode == 2
    assert cli("frobnicate").returncode == 2
    r = cli("solve", "--rhs", "x.csv")
    assert r.returncode == 2 and "--matrix and --rhs are required" in r.stderr
    assert cli("build").returncode == 2
    assert cli("solve", "--matrix").returncode == 2
    r = cli("solve", "--matrix", tmp_path / "a.mtx", "--rhs", tmp_path / "missing.csv")
    assert r.returncode == 3 and r.stderr.startswith("io error: cannot open file for reading")
    spit(tmp_path / "bad.csv", "1\n2\nzz\n")
    r = cli("solve", "--matrix", tmp_path / "a.mtx", "--rhs", tmp_path / "bad.csv")
    assert r.returncode == 3 and "line 3" in r.stderr
    r = cli("build", "--config", tmp_path / "missing.cfg")
    assert r.returncode == 3 and "cannot open config file" in r.stderr


# ------------------------------------------------------------------ Matrix Market (device)
@pytest.mark.gpu
def test_matrix_market_roundtrip_example1(tmp_path, pins):
    d = np.array(pins["example1"]["matrix"], float)
    a = P.Matrix.dense(d)
    path = str(tmp_path / "a.mtx")
    P.write_matrix_market(a, path)
    back = P.read_matrix_market(path)
    assert back.shape == (4, 6)
    assert np.array_equal(back.to_dense(), d)


@pytest.mark.gpu
def test_matrix_market_all_zero(tmp_path):
    a = P.Matrix.from_triplets(5, 8, [], [], [])
    path = str(tmp_path / "zero.mtx")
    P.write_matrix_market(a, path)
    back = P.read_matrix_market(path)
    assert back.shape == (5, 8) and back.stored == 0


@pytest.mark.gpu
def test_matrix_market_byte_stable(tmp_path):
    rng = np.random.default_rng(5001)
    p1, p2 = str(tmp_path / "m1.mtx"), str(tmp_path / "m2.mtx")
    for _ in range(10):
        m, n = int(rng.integers(1, 31)), int(rng.integers(1, 31))
        mask = rng.uniform(size=(m, n)) < 0.3
        r, c = np.nonzero(mask)
        v = rng.uniform(-1e6, 1e6, len(r))
        a = P.Matrix.from_triplets(m, n, r, c, v)
        P.write_matrix_market(a, p1)
        P.write_matrix_market(P.read_matrix_market(p1), p2)
        b1, b2 = open(p1, "rb").read(), open(p2, "rb").read()
        assert b1 == b2
        order = np.lexsort((c, r))
        ptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=m))])
        assert b1 == mm_bytes(m, n, ptr, c[order], v[order])


@pytest.mark.gpu
def test_matrix_market_explicit_zero_kept_on_read_dropped_on_write(tmp_path):
    path = str(tmp_path / "z.mtx")
    spit(path, "%%MatrixMarket matrix coordinate real general\n% comment\n\n2 3 2\n"
               "2 3 0.0\n1 1 4.5\n")
    a = P.read_matrix_market(path)
    assert a.shape == (2, 3) and a.stored == 2 and a.nonzeros() == 1
    P.write_matrix_market(a, path)
    assert open(path).read() == ("%%MatrixMarket matrix coordinate real general\n2 3 1\n"
                                 "1 1 4.5\n")


@pytest.mark.gpu
def test_matrix_market_rejects_malformed_input(tmp_path):
    path = str(tmp_path / "bad.mtx")
    cases = [
        ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
         "line 1: expected '%%MatrixMarket matrix coordinate real general'"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 5.0\n",
         r"line 3: index \(3,1\) out of range for 2x2"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 5.0\n1 1 6.0\n",
         r"line 4: duplicate entry \(1,1\)"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nope\n",
         "line 3: not a number: 'nope'"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1.5 1 2\n",
         "line 3: not an integer index: '1.5'"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 2\n",
         "entry count 1 does not match declared 2"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n",
         "line 3: non-finite value"),
        ("%%MatrixMarket matrix coordinate real general\nfoo\n", "line 2: malformed size line"),
        ("%%MatrixMarket matrix coordinate real general\n% only\n", "missing size line"),
        ("", "empty Matrix Market file"),
    ]
    for text, msg in cases:
        spit(path, text)
        with pytest.raises(P.IoError, match=msg):
            P.read_matrix_market(path)
    with pytest.raises(P.IoError, match="cannot open file for reading"):
        P.read_matrix_market(str(tmp_path / "missing.mtx"))


# ------------------------------------------------------------------ CLI build / solve (device)
@pytest.fixture(scope="module")
def cfg1_files(tmp_path_factory):
    d = tmp_path_factory.mktemp("cli")
    w = CONFIGS[1]
    spit(d / "scan.cfg", config_text(w))
    r = cli("build", "--config", d / "scan.cfg", "--out-matrix", d / "a.mtx",
            "--phantom", "shepp-logan", "--out-rhs", d / "p.csv", "--json")
    assert r.returncode == 0, r.stderr
    return d, w, json.loads(r.stdout)


@pytest.mark.gpu
def test_cli_build_matches_oracle(cfg1_files):
    d, w, rep = cfg1_files
    _, cfg, a, csr, _, _ = oracle_workload(1)
    rows, cols, _ = csr.info()
    ptr, idx, val = csr.arrays()
    assert rep["rows"] == rows == w.m and rep["cols"] == cols == w.n and rep["symmetric"]
    assert open(d / "a.mtx", "rb").read() == mm_bytes(rows, cols, ptr, idx, val)
    p_ref = O.forward_project_csr(csr, O.rasterize(O.shepp_logan(), O.make_grid(cfg)))
    p = P.read_vector_csv(str(d / "p.csv"))
    assert p.tobytes() == p_ref.tobytes()
    s = O.split_system(a, p_ref, 0.0)
    assert rep["fill1"] == s.fill1 and rep["fill2"] == s.fill2


@pytest.mark.gpu
def test_cli_solve_split_matches_api_and_oracle(cfg1_files, tmp_path):
    d, w, _ = cfg1_files
    out = tmp_path / "f.csv"
    r = cli("solve", "--matrix", d / "a.mtx", "--rhs", d / "p.csv", "--mode", "split",
            "--method", "sart", "--tol", 0, "--max-iters", w.iters, "--relaxation",
            w.relaxation, "--sym-tol", 0, "--out", out, "--json")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["method"] == "sart" and rep["mode"] == "split" and rep["iterations"] == w.iters
    assert len(rep["branch_seconds"]) == 2
    f_cli = P.read_vector_csv(str(out))
    sys_ = P.CentroSystem(P.read_matrix_market(str(d / "a.mtx")),
                          P.read_vector_csv(str(d / "p.csv")), 0.0)
    api = P.solve_split(sys_, P.SolveOptions(max_iters=w.iters, tol=0.0,
                                              relaxation=w.relaxation))
    assert f_cli.tobytes() == api.f.tobytes()
    _, cfg, a, _, _, _ = oracle_workload(1)
    p_ref = P.read_vector_csv(str(d / "p.csv"))
    ref = O.solve_split(a, p_ref, 0.0, w.iters, 0.0, w.relaxation)
    assert np.linalg.norm(f_cli - ref.f) <= 1e-10 * np.linalg.norm(ref.f)


@pytest.mark.gpu
def test_cli_parallel_flag_is_deterministic(cfg1_files, tmp_path):
    """acceptance.cpp:382-420 (criterion 9): --parallel 1 and 8 give identical bytes."""
    d, w, _ = cfg1_files
    outs = []
    for par in (1, 8):
        out = tmp_path / ("f%d.csv" % par)
        r = cli("solve", "--matrix", d / "a.mtx", "--rhs", d / "p.csv", "--mode", "split",
                "--method", "cgls", "--sym-tol", 0, "--max-iters", 20, "--parallel", par,
                "--out", out)
        assert r.returncode == 0, r.stderr
        assert r.stdout.startswith("method=cgls mode=split iterations=")
        outs.append(open(out, "rb").read())
    assert outs[0] and outs[0] == outs[1]


@pytest.mark.gpu
def test_cli_split_rejects_asymmetric_matrix(tmp_path):
    path = str(tmp_path / "asym.mtx")
    spit(path, "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n")
    P.write_vector_csv([1.0, 2.0], str(tmp_path / "p.csv"))
    r = cli("solve", "--matrix", path, "--rhs", tmp_path / "p.csv", "--mode", "split")
    sym = P.verify_symmetry(P.read_matrix_market(path), 1e-12)
    assert r.returncode == 1
    assert ("split mode needs a centrosymmetric matrix: max violation %g at (%d,%d) exceeds tol "
            "1e-12" % (sym.max_violation, sym.worst_row, sym.worst_col)) in r.stderr
    assert sym.max_violation == 1.0
    r = cli("solve", "--matrix", path, "--rhs", tmp_path / "p.csv", "--method", "nope")
    assert r.returncode == 1 and "unknown method name" in r.stderr
    P.write_vector_csv([1.0], str(tmp_path / "short.csv"))
    r = cli("solve", "--matrix", path, "--rhs", tmp_path / "short.csv")
    assert r.returncode == 1 and "rhs length does not match" in r.stderr
