"""The maintainer's ``mode="gpu"`` patch of the reference,
applied to a COPY of the installed reference (``oracle/_ref/gsmat``) so the
reference's own test modules can run against the drop-in
(tests/test_reference_suite.py).  Test infrastructure: nothing here is
imported by the product.

The snippets below are the ones INTEGRATION.md §2 prints (a CPU test checks
that the document carries them verbatim).
"""

from __future__ import annotations

import shutil
from pathlib import Path

# gsmat/executor.py, at the top of execute() (executor.py:310): route "gpu"
# -- and, with GSMAT_DEVICE=gpu, every mode -- to the B200 executor; the
# "sequential"/"parallel" budget rules are kept per mode, "gpu" applies the
# sequential (emitted rows) rule.
EXECUTOR_PATCH = '''\
    if mode == "gpu" or os.environ.get("GSMAT_DEVICE") == "gpu":
        import paper_1807_07691_b200 as _b200
        from . import errors as _errors
        try:
            return _b200.execute(query, plan, store, mode=mode, worker_count=worker_count,
                                 row_budget=row_budget, report=report)
        except _b200.GsmatError as exc:
            raise _b200.errors.as_reference_error(exc, _errors) from None
'''
EXECUTOR_ANCHOR = '    if mode not in ("sequential", "parallel"):\n        raise ValueError(f"unknown mode {mode!r}")\n'

# gsmat/cli.py:40: the CLI's --mode accepts "gpu"
CLI_OLD = 'p.add_argument("--mode", choices=["sequential", "parallel"], default=None)'
CLI_NEW = 'p.add_argument("--mode", choices=["sequential", "parallel", "gpu"], default=None)'


def apply(installed_pkg: Path, dst: Path) -> Path:
    """Copy ``installed_pkg`` (a ``gsmat`` package directory) to ``dst/gsmat``
    and apply the patch; returns the patched package directory."""
    out = dst / "gsmat"
    shutil.copytree(installed_pkg, out)
    ex = out / "executor.py"
    text = ex.read_text()
    assert text.count(EXECUTOR_ANCHOR) == 1, "reference execute() changed; patch anchor not found"
    text = text.replace(EXECUTOR_ANCHOR, EXECUTOR_PATCH + EXECUTOR_ANCHOR)
    text = text.replace("import time\n", "import os\nimport time\n", 1)
    ex.write_text(text)
    cli = out / "cli.py"
    text = cli.read_text()
    assert text.count(CLI_OLD) == 1, "reference cli changed; patch anchor not found"
    cli.write_text(text.replace(CLI_OLD, CLI_NEW))
    for pyc in out.rglob("__pycache__"):
        shutil.rmtree(pyc)
    return out
