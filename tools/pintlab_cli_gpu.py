"""Run the reference's own CLI (``pintlab.cli``) on the B200 path.

    PYTHONPATH=/path/to/pintlab/src python tools/pintlab_cli_gpu.py single-run --set dim=3 ...

The reference's experiment drivers import ``Grid``, ``HeatOperator``,
``Level``, ``MgConfig``, ``pfasst_run``, ``run_sdc`` ... from its own modules.
This launcher registers this package's modules under the reference's module
names for exactly the accelerated path (heat, transfers, multigrid,
quadrature, sdc, hierarchy, pfasst) and then hands ``sys.argv`` to the
reference's ``cli.main`` unchanged: configuration parsing, presets, CSV
writing and the footer are the reference's own code (not restated here).
``--set executor=nccl`` is accepted once ``config.EXECUTORS`` allows it; the
launcher widens that tuple for the run (the one-line change INTEGRATION.md
section 4 shows for a maintainer).  Requires the reference package on
PYTHONPATH; nothing here is used by the tests or the benchmark.
"""
from __future__ import annotations

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ACCELERATED = ("heat", "transfers", "multigrid", "quadrature", "sdc", "hierarchy", "pfasst")


def install():
    import pintlab  # noqa: F401  (the reference package itself)
    for name in ACCELERATED:
        sys.modules[f"pintlab.{name}"] = importlib.import_module(f"paper_1407_6486_b200.{name}")
    config = importlib.import_module("pintlab.config")
    if "nccl" not in config.EXECUTORS:
        config.EXECUTORS = tuple(config.EXECUTORS) + ("nccl",)
    return importlib.import_module("pintlab.cli")


if __name__ == "__main__":
    sys.exit(install().main(sys.argv[1:]))
