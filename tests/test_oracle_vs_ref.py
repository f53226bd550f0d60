"""Differential pinning of the oracle against the UNMODIFIED reference
(oracle/_ref/libjsontape_ref.so, built from /root/reference by
oracle/build_ref.sh).  Skipped where the prebuilt reference is absent."""
import os
import random

import pytest

from oracle.pyoracle import REF_SO
from tests.test_gpu_parity import _mutate, _rand_json
from tests.test_kernels_cpu import _rand_number
from tests.vectors import SOUP_POOL

pytestmark = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    from oracle.pyoracle import Reference
    return Reference()


def _same(oracle, ref, d):
    a, b = oracle.parse(d), ref.parse(d)
    assert (a.code, a.offset) == (b.code, b.offset), d[:120]
    if b.code != 1:
        assert a.index == b.index, d[:120]
    if b.code == 0:
        assert a.tape == b.tape and a.strings == b.strings, d[:120]


def test_soup(oracle, ref):
    # test_indexer.cpp:73-81 pool
    rng = random.Random(17)
    for _ in range(3000):
        _same(oracle, ref, bytes(rng.choice(SOUP_POOL) for _ in range(rng.randrange(0, 1500))))


def test_random_json_and_mutations(oracle, ref):
    rng = random.Random(29)
    for _ in range(2000):
        d = _rand_json(rng).encode()
        _same(oracle, ref, d)
        _same(oracle, ref, _mutate(rng, d))


def test_numbers(oracle, ref):
    rng = random.Random(31)
    for _ in range(20000):
        t = _rand_number(rng)
        _same(oracle, ref, b"[" + t + b"]")


def test_configs(oracle, ref):
    from tools.gen import generate
    for cfg, size in [(0, 1 << 18), (1, 1 << 19), (2, 1 << 19), (4, 1 << 19)]:
        _same(oracle, ref, generate(cfg, size))
    for rec in generate(3, 1 << 18).split(b"\n")[:500]:
        _same(oracle, ref, rec)
    for seed in range(1, 100):
        _same(oracle, ref, generate(4, 1 << 13, seed=seed, err=1 + seed % 5))


def test_minify(oracle, ref):
    """jt_minify (capi.cpp:154-167, minify_pass indexer.cpp:58-75): the
    oracle's restatement against the reference on valid and invalid input"""
    from tools.gen import generate
    rng = random.Random(41)
    docs = [b' { "a" : [ 1 , "x y\\" z" ] } ', b"[1,]", b'{"k": "\\\\", "v": [true, null]}\n', b"",
            generate(1, 1 << 18), generate(4, 1 << 17), generate(0, 1 << 16)]
    for _ in range(1500):
        d = _rand_json(rng).encode()
        docs += [d, _mutate(rng, d)]
    for d in docs:
        assert oracle.minify(d) == ref.minify(d), d[:120]


def test_stats(oracle, ref):
    """jt_compute_stats restatement (oracle) against the reference"""
    from tools.gen import generate
    rng = random.Random(47)
    docs = [generate(0, 1 << 16), generate(1, 1 << 17), b"[1, 2.5, \"x\", {}, [], null, true, false]",
            b"[1,]", b""]
    for _ in range(300):
        d = _rand_json(rng).encode()
        docs += [d, _mutate(rng, d)]
    for d in docs:
        assert oracle.stats(d) == ref.stats(d), d[:120]
