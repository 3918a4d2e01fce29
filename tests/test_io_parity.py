"""CPU: the drop-in's file API (include/chainhull/io.hpp over
paper_1508_05488_b200/cpp/chainhull_io.cpp) against the reference's own
io.cpp (io.cpp:38-261): tests/io_probe.cpp is built against each
(build/io_probe_b200, oracle/_ref/io_probe_ref) and must print the same
lines (read results, error types, line numbers and messages) and write the
same bytes (xy_text at 17 significant digits, xy_binary, hull text, stats
CSV and JSON)."""
import filecmp
import os
import subprocess

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "oracle", "_ref", "io_probe_ref")
OURS = os.path.join(ROOT, "build", "io_probe_b200")


@pytest.mark.skipif(not (os.path.exists(REF) and os.path.exists(OURS)),
                    reason="io probes not built (make; make -C oracle)")
def test_io_byte_parity(tmp_path):
    a, b = tmp_path / "ref", tmp_path / "ours"
    ra = subprocess.run([REF, str(a)], capture_output=True, text=True, timeout=120)
    rb = subprocess.run([OURS, str(b)], capture_output=True, text=True, timeout=120)
    assert ra.returncode == 0 and rb.returncode == 0, (ra.stderr, rb.stderr)
    assert ra.stdout == rb.stdout
    names = sorted(os.listdir(a))
    assert names == sorted(os.listdir(b)) and len(names) >= 13
    for n in names:
        assert filecmp.cmp(a / n, b / n, shallow=False), n
