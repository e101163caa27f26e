"""The C-ABI library builds/loads and exports every symbol include/be200.h declares."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "be200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(be_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    from paper_2401_07886_b200 import _lib
    lib = _lib.load()
    names = declared()
    assert "be_rollout_greedy" in names and "be_reduce_eval" in names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)
    assert lib.be_abi_version() == 1


def test_struct_sizes_match_c():
    from paper_2401_07886_b200 import _lib
    # be_tier 32 B; be_cfg layout checked against offsets in the header
    assert ctypes.sizeof(_lib.BeTier) == 32
    assert ctypes.sizeof(_lib.BeTraceSoa) == 16 + 8 * 8 + 2 * 4  # + env_ready, envs_per_ready, ready_value
    assert ctypes.sizeof(_lib.BeQWeights) == 8 + 4 * 8
    assert ctypes.sizeof(_lib.BeRecords) == 6 * 8
    assert ctypes.sizeof(_lib.BeGenCfg) == 128
    assert ctypes.sizeof(_lib.BeThresholds) == 8 + 8 * _lib.MAX_THETA  # be_thresholds, by value
    assert ctypes.sizeof(_lib.BeTrainIterCfg) == 3 * 8 + 2 * 8 + 8 + 6 * 4  # ... use_gate, router, _pad
