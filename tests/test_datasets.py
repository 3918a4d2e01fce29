"""CPU: the generator behind the benchmark and the sharded run
(paper_1508_05488_b200/csrc/datasets.cpp). generate() must equal the
reference's own generate() (datasets.cpp:94-106) and any slice
generate(begin, count) must equal the same rows of the whole set, so that
each rank of the sharded 1B run holds exactly its contiguous shard."""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_1508_05488_b200 as P  # noqa: E402
from pyoracle import DISTRIBUTIONS, Oracle, RefLib  # noqa: E402


@pytest.mark.parametrize("dist", DISTRIBUTIONS)
def test_generate_matches_reference(dist):
    ref = RefLib() if RefLib.available() else Oracle()
    for n, seed in ((1, 3), (1000, 42), (4097, 7)):
        assert np.array_equal(P.generate(dist, n, seed), ref.generate(dist, n, seed)), (dist, n)


@pytest.mark.parametrize("dist", DISTRIBUTIONS)
def test_generate_range_is_a_slice(dist):
    n, seed = 10_000, 11
    whole = P.generate(dist, n, seed)
    for begin, count in ((0, n), (0, 1), (1, 1), (3333, 4000), (n - 1, 1), (n, 0), (5000, 5000)):
        part = P.generate(dist, n, seed, begin=begin, count=count)
        assert part.shape == (count, 2)
        assert np.array_equal(part.view(np.uint64), whole[begin:begin + count].view(np.uint64))


def test_generate_range_contiguous_shards_cover_the_set():
    n, seed, world = 50_001, 42, 4
    whole = P.generate("uniform_square", n, seed)
    bounds = [n * r // world for r in range(world + 1)]
    parts = [P.generate("uniform_square", n, seed, begin=bounds[r], count=bounds[r + 1] - bounds[r])
             for r in range(world)]
    assert np.array_equal(np.concatenate(parts), whole)


def test_generate_range_rejects_bad_slices():
    with pytest.raises(ValueError):
        P.generate("uniform_square", 10, 1, begin=8, count=3)
    out = np.empty((4, 2))
    P.generate("gaussian", 10, 1, begin=2, count=4, out=out)
    assert np.array_equal(out, P.generate("gaussian", 10, 1)[2:6])
