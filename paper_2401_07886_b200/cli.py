"""`--backend b200` for the reference command line (the
reference CLI is pkg/src/besteffort/cli.py).

The reference CLI (gen / train / finetune / eval / report) stays the front end:
argument parsing, config, seeds, checkpoint and CSV writers, exit codes.  This
module only swaps its three compute entry points for the GPU drop-ins before
handing over to the reference's own `main`:

  besteffort.cli.run_eval      -> paper_2401_07886_b200.run_eval      (cli.py:179-186)
  besteffort.cli.run_training  -> paper_2401_07886_b200.trainer.run_training (cli.py:115)
  besteffort.cli.fine_tune     -> paper_2401_07886_b200.trainer.fine_tune    (cli.py:136)

so `eval` writes byte-identical metrics / summary / per-rate files (the
records are bit-identical, tests/test_cli_backend_gpu.py) and `train` /
`finetune` write reference-format BEQN1 checkpoints and train logs.

usage:  python -m paper_2401_07886_b200.cli [--backend b200|reference] <reference CLI args>
The reference package must be importable (e.g. PYTHONPATH=baseline/_ref).
"""
from __future__ import annotations

import sys
from typing import Optional

BACKENDS = ("b200", "reference")


def install(cli_module) -> None:
    """Point a reference CLI module's compute entry points at the GPU path."""
    from .evalkit import run_eval
    from .trainer import fine_tune, run_training
    cli_module.run_eval = run_eval
    cli_module.run_training = run_training
    cli_module.fine_tune = fine_tune


def split_backend(argv: list) -> tuple:
    """(backend, remaining argv): `--backend X` / `--backend=X` anywhere in argv."""
    backend, rest, i = "b200", [], 0
    while i < len(argv):
        a = argv[i]
        if a == "--backend":
            if i + 1 >= len(argv):
                raise ValueError("--backend needs a value")
            backend = argv[i + 1]
            i += 2
            continue
        if a.startswith("--backend="):
            backend = a.split("=", 1)[1]
        else:
            rest.append(a)
        i += 1
    if backend not in BACKENDS:
        raise ValueError(f"--backend must be one of {', '.join(BACKENDS)}")
    return backend, rest


def main(argv: Optional[list] = None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    try:
        backend, rest = split_backend(argv)
    except ValueError as e:  # the reference CLI's convention: usage errors exit 2
        print(f"error: {e}", file=sys.stderr)
        return 2
    import besteffort.cli as ref_cli
    if backend == "b200":
        install(ref_cli)
    return ref_cli.main(rest)


if __name__ == "__main__":
    sys.exit(main())
