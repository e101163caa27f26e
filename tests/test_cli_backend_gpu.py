"""The reference command line with `--backend b200` (paper_2401_07886_b200/cli.py,
SURVEY.md §8f-2): `eval` writes byte-identical metrics / summary / per-rate
CSVs to the reference backend's (cli.py:163-216); `train` / `finetune` write
BEQN1 checkpoints the reference loads and reference-format train logs.  Each
backend runs in its own process, as a user would invoke it.  Needs the
reference package in baseline/_ref (skipped otherwise)."""
import hashlib
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
POLICY = os.path.join(ROOT, "tests", "golden", "trained_seed7.beqn")

pytestmark = pytest.mark.gpu


def _cli(args, out, backend):
    if not os.path.isdir(os.path.join(REF, "besteffort")):
        pytest.skip("reference package not installed in baseline/_ref")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]), OPENBLAS_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "paper_2401_07886_b200.cli", "--backend", backend] + args + ["--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    return r


def _digests(d):
    return {f: hashlib.sha256(open(os.path.join(d, f), "rb").read()).hexdigest() for f in sorted(os.listdir(d))}


@pytest.mark.parametrize("scenario,policy", [("stable", POLICY), ("unpredictable-1", POLICY),
                                             ("hellaswag-copa-soft", "static:1")])
def test_eval_outputs_byte_identical(cuda, tmp_path, scenario, policy):
    out = {}
    for b in ("reference", "b200"):
        d = tmp_path / b
        r = _cli(["eval", "--scenario", scenario, "--policy", policy, "--seed", "3"], d, b)
        assert r.returncode == 0, r.stderr[-2000:]
        out[b] = _digests(d)
    assert out["b200"] and out["b200"] == out["reference"]


def test_train_and_finetune_write_reference_checkpoints(cuda, tmp_path):
    sys.path.insert(0, REF)
    r = _cli(["train", "--iterations", "3000", "--seed", "1"], tmp_path, "b200")
    assert r.returncode == 0, r.stderr[-2000:]
    ckpt = tmp_path / "policy_base_seed1.bqn"
    log = tmp_path / "train_log_base_seed1.csv"
    assert ckpt.exists() and log.exists()
    assert open(log).readline().strip() == "step,loss,mean_recent_reward,epsilon"
    from besteffort.policy import load_checkpoint
    net = load_checkpoint(str(ckpt), n_tasks=4, n_tiers=3)
    assert net.hidden == 256
    r = _cli(["finetune", "--policy", str(ckpt), "--iterations", "2000", "--seed", "2"], tmp_path, "b200")
    assert r.returncode == 0, r.stderr[-2000:]
    assert (tmp_path / "policy_soft_finetuned_seed2.bqn").exists()


def test_usage_errors_exit_2(cuda, tmp_path):
    r = _cli(["eval", "--scenario", "no-such-scenario", "--policy", "static:0"], tmp_path, "b200")
    assert r.returncode == 2
    r = _cli(["eval", "--scenario", "stable", "--policy", "static:7"], tmp_path, "b200")
    assert r.returncode == 2 and "out of range" in r.stderr
