"""The reference command line (proj/tools/src/main.cpp) over the drop-in:
build/chainhull (paper_1508_05488_b200/tools/chainhull_cli.cpp).

Mirrors the reference's own CLI tests (proj/tests/cli_test.cpp: exit codes,
end-to-end hull, chunk-count invariance, verify, bench rows) and pins the
bench CSV schema of main.cpp:159-161 byte for byte. CPU tests cover what
runs before any device work (usage errors, gen, malformed input); the
`gpu` tests run the hull path and compare the CSV counters with the
reference's own convex_hull (oracle/_ref) on the same inputs.
"""
import csv
import io
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CLI = os.path.join(ROOT, "build", "chainhull")
HEADER = ("size,seed,repeat,n_input,n_after_round1,n_after_spa,n_hull,t_extremes_ms,"
          "t_classify_ms,t_partition_ms,t_sort_ms,t_spa_ms,t_melkman_ms,t_total_ms,"
          "frac_after_round1,frac_after_spa")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="build/chainhull not built (make)")


def run(*args, env=None):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600,
                          env=env)


def reflib():
    from pyoracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    return RefLib()


# ------------------------------------------------------------------ CPU

def test_usage_errors_exit_2(tmp_path):
    # cli_test.cpp:66-72
    assert run("hull", "--input", tmp_path / "missing.xy", "--output", tmp_path / "h.xy").returncode == 2
    assert run("verify", "--n", 100, "--trials", 0).returncode == 2
    assert run("gen", "--n", 10, "--output", tmp_path / "g.xy",
               "--distribution", "no_such").returncode == 2
    assert run("--help").returncode == 0
    assert run().returncode == 2
    assert run("bench").returncode == 2                       # --sizes is required
    assert run("bench", "--sizes", "10,x").returncode == 2
    assert run("hull", "--bogus", 1).returncode == 2
    assert run("verify", "--trials", 2).returncode == 2        # needs --input or --n
    assert run("frobnicate").returncode == 2


def test_malformed_input_is_a_runtime_error(tmp_path):
    # cli_test.cpp:74-80: malformed content exits 1, not 2
    bad = tmp_path / "bad.xy"
    bad.write_text("zero zero\n")
    r = run("hull", "--input", bad, "--output", tmp_path / "h.xy")
    assert r.returncode == 1
    assert "line 1" in r.stderr


@pytest.mark.parametrize("fmt", ["xy_text", "xy_binary"])
@pytest.mark.parametrize("dist", ["uniform_square", "uniform_disk", "gaussian", "circle"])
def test_gen_matches_reference_generator(tmp_path, fmt, dist):
    ref = reflib()
    out = tmp_path / "g"
    r = run("gen", "--distribution", dist, "--n", 777, "--seed", 5, "--output", out, "--format", fmt)
    assert r.returncode == 0, r.stderr
    assert r.stdout == f"gen: 777 {dist} points -> {out}\n"
    want = ref.generate(dist, 777, 5)
    if fmt == "xy_binary":
        got = np.fromfile(out, dtype="<f8").reshape(-1, 2)
    else:
        got = np.loadtxt(out).reshape(-1, 2)
    assert got.tobytes() == want.tobytes()


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_hull_end_to_end(tmp_path):
    # cli_test.cpp:52-63
    sq = tmp_path / "square.xy"
    sq.write_text("0 0\n1 0\n1 1\n0 1\n0.5 0.5\n0.25 0.75\n")
    r = run("hull", "--input", sq, "--output", tmp_path / "hull.xy",
            "--stats-output", tmp_path / "stats.csv")
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "hull.xy").read_text() == "0 0\n1 0\n1 1\n0 1\n"
    assert (tmp_path / "stats.csv").read_text().startswith("n_input,")
    r = run("hull", "--input", sq, "--output", tmp_path / "hull2.xy",
            "--stats-output", tmp_path / "stats.json", "--stats-format", "json")
    assert r.returncode == 0 and (tmp_path / "stats.json").read_text().startswith("{\n")


@pytest.mark.gpu
def test_hull_identical_for_every_chunk_count(tmp_path):
    # cli_test.cpp:83-95, plus the bytes of the reference's hull
    pts = tmp_path / "pts.xy"
    assert run("gen", "--distribution", "uniform_disk", "--n", 20000, "--seed", 5,
               "--output", pts).returncode == 0
    outs = []
    for c in (1, 7, 1024):
        assert run("hull", "--input", pts, "--chunk-count", c, "--output",
                   tmp_path / f"h{c}.xy").returncode == 0
        outs.append((tmp_path / f"h{c}.xy").read_text())
    assert outs[0] == outs[1] == outs[2] and outs[0]
    ref = reflib()
    want = ref.convex_hull(ref.generate("uniform_disk", 20000, 5), 1024)[0].hull
    assert np.loadtxt(io.StringIO(outs[0])).tobytes() == want.tobytes()


@pytest.mark.gpu
def test_verify_agrees_with_the_reference_hull():
    # cli_test.cpp:97-104
    r = run("verify", "--distribution", "uniform_square", "--n", 2000, "--trials", 3,
            "--chunk-counts", 1, 1024)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.splitlines()[-1] == "verified 3/3 trials"
    assert r.stdout.splitlines()[0].startswith("trial 0 seed=0 n=2000 n_hull=")
    assert run("verify", "--distribution", "uniform_disk", "--n", 1000, "--trials", 2,
               "--chunk-counts", "1,16,1024").returncode == 0
    assert run("verify", "--distribution", "collinear", "--n", 500, "--trials", 2).returncode == 0
    assert run("verify", "--distribution", "circle", "--n", 3000, "--seed", 9).returncode == 0


@pytest.mark.gpu
def test_bench_rows_and_schema(tmp_path):
    # cli_test.cpp:106-113 and the header of main.cpp:159-161
    out = tmp_path / "bench.csv"
    r = run("bench", "--sizes", 1000, 2000, "--seeds", 1, 2, "--repeats", 2, "--csv-output", out)
    assert r.returncode == 0, r.stderr
    text = out.read_text()
    assert text.startswith(HEADER + "\n")
    assert text.count("\n") == 9  # header + 8 rows
    r = run("bench", "--sizes", "3000,20000", "--distribution", "gaussian", "--seeds", 4,
            "--with-oracle")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert r.stdout.splitlines()[0] == HEADER + ",t_oracle_ms"
    ref = reflib()
    for row in rows:
        n, seed = int(row["size"]), int(row["seed"])
        h, _ = ref.convex_hull(ref.generate("gaussian", n, seed), 1024)
        assert [int(row[k]) for k in ("n_input", "n_after_round1", "n_after_spa", "n_hull")] \
            == [int(c) for c in h.counts]
        assert row["frac_after_spa"] == "%.6f" % (int(row["n_after_spa"]) / n)
        for k in ("t_extremes_ms", "t_total_ms", "t_oracle_ms"):
            assert float(row[k]) >= 0.0 and len(row[k].split(".")[1]) == 6
