"""The cprand_b200 front end (tools/cprand_b200_cli.cpp): the reference's
decompose / bench-iter commands (tools/cprand_main.cpp:134-206) over DNT1
files (io.hpp:20-87), writing the model JSON (io.hpp:89-142) and the trace
CSV (io.hpp:144-153). CPU tests: usage, file-format and exit-code
behaviour; GPU tests: a decompose run against the oracle."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "cprand_b200")
sys.path.insert(0, os.path.join(ROOT, "oracle"))


@pytest.fixture(scope="module")
def cli():
    subprocess.check_call(["make", "-s", "-C", ROOT, "cli"])
    assert os.path.exists(CLI)
    return CLI


def write_dnt1(path, x):
    """DNT1: magic, u64 order, u64 dims, f64 values in storage order (mode-1 fastest)."""
    with open(path, "wb") as f:
        f.write(b"DNT1")
        f.write(struct.pack("<Q", x.ndim))
        for d in x.shape:
            f.write(struct.pack("<Q", d))
        f.write(np.asarray(x, dtype="<f8").reshape(-1, order="F").tobytes())


def run(cli, *args):
    p = subprocess.run([cli, *args], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


def test_usage_and_argument_errors(cli, tmp_path):
    assert run(cli, "--help")[0] == 0
    assert run(cli)[0] == 2
    rc, _, err = run(cli, "decompose", "--rank", "3")
    assert rc == 2 and "--in is required" in err
    rc, _, err = run(cli, "decompose", "--in", "x", "--rank", "3", "--out", "m", "--bogus", "1")
    assert rc == 2 and "unknown option" in err
    rc, _, err = run(cli, "gen", "--out", "x")
    assert rc == 2 and "not on the B200 path" in err
    rc, _, err = run(cli, "eval", "--in", "x")
    assert rc == 2 and "--model is required" in err


def test_dnt1_reader_rejects_bad_files(cli, tmp_path):
    bad = tmp_path / "bad.dnt"
    bad.write_bytes(b"NOPE")
    rc, _, err = run(cli, "decompose", "--in", str(bad), "--rank", "2", "--method", "rand", "--out", str(tmp_path / "m"))
    assert rc == 2 and "not a DNT1 tensor file" in err
    trunc = tmp_path / "trunc.dnt"
    x = np.arange(24, dtype=float).reshape(2, 3, 4)
    write_dnt1(trunc, x)
    trunc.write_bytes(trunc.read_bytes()[:-8])
    rc, _, err = run(cli, "decompose", "--in", str(trunc), "--rank", "2", "--method", "rand", "--out", str(tmp_path / "m"))
    assert rc == 2 and "truncated" in err


@pytest.mark.gpu
@pytest.mark.parametrize("method,transform", [("rand", None), ("mix", "dct"), ("mix", None)])
def test_decompose_matches_oracle(cli, tmp_path, method, transform):
    import oracle as orc
    x, _ = orc.gen_baseline((20, 18, 16), 3, 0.5, 0.01, 4)
    f = tmp_path / "x.dnt"
    write_dnt1(f, x)
    args = ["decompose", "--in", str(f), "--method", method, "--rank", "3", "--samples", "60", "--seed", "4",
            "--max-iters", "25", "--stall", "1000", "--fit-samples", "2048", "--out", str(tmp_path / "m.json"),
            "--trace", str(tmp_path / "t.csv")]
    if transform:
        args += ["--transform", transform]
    rc, out, err = run(cli, *args)
    assert rc == 0, err
    kv = dict(p.split("=", 1) for p in out.split())
    ref = orc.solve(method, x, 3, 60, orc.SolveOptions(rng_seed=4, max_iters=25, stall_limit=1000,
                                                        fit_sample_count=2048, transform=transform))
    assert kv["method"] == method and int(kv["iters"]) == ref.iterations == 25
    assert kv["stop"] == "max_iterations"
    assert abs(float(kv["fit"]) - ref.trace[-1][2]) < 1e-8
    model = json.loads((tmp_path / "m.json").read_text())
    assert len(model["factors"]) == 3 and len(model["lambda"]) == 3
    for got, want in zip(model["factors"], ref.factors):
        got = np.array(got)
        assert got.shape == want.shape
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-6
    lines = (tmp_path / "t.csv").read_text().strip().split("\n")
    assert lines[0] == "iter,time_s,fit,fit_kind,best_fit" and len(lines) == 26
    it, _, fit, kind, _ = lines[-1].split(",")
    assert int(it) == 25 and kind == "estimated" and abs(float(fit) - ref.trace[-1][2]) < 1e-8


@pytest.mark.gpu
def test_bench_iter_csv(cli, tmp_path):
    import oracle as orc
    x = orc.random_tensor((24, 20, 16), 3)
    f = tmp_path / "x.dnt"
    write_dnt1(f, x)
    rc, out, err = run(cli, "bench-iter", "--in", str(f), "--rank", "4", "--method", "rand", "--method", "mix",
                       "--transform", "dct", "--iters", "20")
    assert rc == 0, err
    lines = out.strip().split("\n")
    assert lines[0] == "method,iters,setup_s,mean_iter_s"
    rows = [l.split(",") for l in lines[1:]]
    assert [r[0] for r in rows] == ["rand", "mix"] and all(int(r[1]) == 20 for r in rows)
    assert all(float(r[3]) > 0 for r in rows)
    rc, _, err = run(cli, "bench-iter", "--in", str(f), "--rank", "4", "--method", "als")
    assert rc == 2 and "outside the B200 path" in err


@pytest.mark.gpu
def test_eval_fit_and_score(cli, tmp_path):
    """eval: the exact fit on the GPU and the score against a truth model
    (the decompose output read back through the model JSON reader)."""
    import oracle as orc
    x, truth = orc.gen_baseline((20, 18, 16), 3, 0.3, 0.01, 8)
    f = tmp_path / "x.dnt"
    write_dnt1(f, x)
    rc, _, err = run(cli, "decompose", "--in", str(f), "--method", "rand", "--rank", "3", "--samples", "60",
                     "--seed", "8", "--max-iters", "30", "--out", str(tmp_path / "m.json"))
    assert rc == 0, err
    model = json.loads((tmp_path / "m.json").read_text())
    lam = np.array(model["lambda"])
    fs = [np.array(a) for a in model["factors"]]
    (tmp_path / "t.json").write_text(json.dumps({"lambda": [1.0] * 3, "factors": [a.tolist() for a in truth]}))
    rc, out, err = run(cli, "eval", "--model", str(tmp_path / "m.json"), "--in", str(f),
                       "--truth", str(tmp_path / "t.json"))
    assert rc == 0, err
    kv = dict(l.split(",") for l in out.strip().split("\n"))
    assert abs(float(kv["fit"]) - orc.exact_fit(x, lam, fs)) < 1e-10
    assert abs(float(kv["score"]) - orc.score(fs, truth)) < 1e-12
    # R > 8: the Hungarian matching (synth.hpp:181-185)
    g = np.random.default_rng(5)
    a = [g.standard_normal((d, 10)) for d in (20, 18, 16)]
    b = [g.standard_normal((d, 10)) for d in (20, 18, 16)]
    for name, fs_ in (("a.json", a), ("b.json", b)):
        (tmp_path / name).write_text(json.dumps({"lambda": [1.0] * 10, "factors": [m.tolist() for m in fs_]}))
    rc, out, err = run(cli, "eval", "--model", str(tmp_path / "a.json"), "--in", str(f),
                       "--truth", str(tmp_path / "b.json"))
    assert rc == 0, err
    kv = dict(l.split(",") for l in out.strip().split("\n"))
    assert abs(float(kv["score"]) - orc.score(a, b)) < 1e-12


def test_io_header_round_trips(tmp_path):
    """include/cprand_b200/io.hpp on the CPU: DNT1 and model-JSON round trips
    bit for bit (17 significant digits), malformed inputs rejected."""
    exe = tmp_path / "io_roundtrip"
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-o", str(exe),
                           os.path.join(ROOT, "tests", "cpp", "io_roundtrip.cpp"),
                           "-L", os.path.join(ROOT, "paper_1701_06600_b200"), "-lcprand_b200",
                           "-Wl,-rpath," + os.path.join(ROOT, "paper_1701_06600_b200")])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout + out.stderr
