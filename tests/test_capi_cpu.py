"""The C-ABI library on a CPU-only host: it loads, exports every symbol
include/fastbdt_b200.h declares, and its host-only entry points (numpy's
PCG64 Fisher-Yates subsample, numpy's pairwise sum) match numpy exactly."""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
import os
import re

import numpy as np
import pytest

from paper_1609_06119_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "fastbdt_b200.h")).read()
    return sorted(set(re.findall(r"\b(bb_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib._SIGS, f"{s} has no ctypes signature"
    assert lib.bb_abi_version() == 1


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 127, 128, 129, 1000, 123457])
def test_pairwise_sum_matches_numpy(n):
    a = np.random.default_rng(n).normal(size=n) * 1e3
    assert _lib.lib().bb_pairwise_sum(_lib.ptr(a), n) == float(np.sum(a))


def _bits_to_mask(bits, n):
    return np.unpackbits(bits.view(np.uint8), bitorder="little")[:n].astype(bool)


def test_host_subsample_matches_golden(golden_dir):
    for rec in json.load(open(f"{golden_dir}/masks.json")):
        a, b, T = rec["n_sig"], rec["n_bkg"], rec["trees"]
        if a + b > 300_000:
            continue
        cfg = _lib.FitConfigC(**_lib.pcg_config(rec["seed"]))
        words = (a + b + 31) // 32
        bits = np.zeros(max(1, words) * T, np.uint32)
        _lib.check(_lib.lib().bb_subsample_masks(a, b, rec["rate"], T, C.byref(cfg), _lib.ptr(bits)))
        for t in range(T):
            m = _bits_to_mask(bits[t * words:(t + 1) * words], a + b)
            assert hashlib.sha1(m.tobytes()).hexdigest() == rec["hashes"][t], (rec["seed"], t)


def test_host_subsample_matches_numpy_directly():
    seed, a, b, rate, T = 77, 12_345, 54_321, 0.37, 3
    rng = np.random.Generator(np.random.PCG64(seed))
    cfg = _lib.FitConfigC(**_lib.pcg_config(seed))
    words = (a + b + 31) // 32
    bits = np.zeros(words * T, np.uint32)
    _lib.check(_lib.lib().bb_subsample_masks(a, b, rate, T, C.byref(cfg), _lib.ptr(bits)))
    for t in range(T):
        ref = []
        for nn in (a, b):
            m = np.zeros(nn, bool)
            m[rng.permutation(nn)[:math.floor(rate * nn)]] = True
            ref.append(m)
        np.testing.assert_array_equal(_bits_to_mask(bits[t * words:(t + 1) * words], a + b), np.concatenate(ref))


def test_errors_map_to_valueerror():
    cfg = _lib.FitConfigC(**_lib.pcg_config(0))
    bits = np.zeros(4, np.uint32)
    with pytest.raises(ValueError, match="subsample rate"):
        _lib.check(_lib.lib().bb_subsample_masks(3, 3, 1.5, 1, C.byref(cfg), _lib.ptr(bits)))
