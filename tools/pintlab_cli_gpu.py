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
PYTHONPATH; tests/test_cli_plumbing.py checks the plumbing on CPU.
"""
from __future__ import annotations

import importlib
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ACCELERATED = ("heat", "transfers", "multigrid", "quadrature", "sdc", "hierarchy", "pfasst")


class _Overlay(types.ModuleType):
    """This package's module for the accelerated names, the reference's own
    module for everything off the path (e.g. heat.exact_pde / exact_ode,
    which the CLI's error columns use and this package does not restate)."""

    def __init__(self, ours, theirs):
        super().__init__(theirs.__name__)
        self.__dict__.update({k: v for k, v in vars(theirs).items() if not k.startswith("__")})
        self.__dict__.update({k: v for k, v in vars(ours).items() if not k.startswith("__")})
        self.__accelerated__ = ours


def install():
    import pintlab  # noqa: F401  (the reference package itself)
    for name in ACCELERATED:
        theirs = importlib.import_module(f"pintlab.{name}")
        ours = importlib.import_module(f"paper_1407_6486_b200.{name}")
        sys.modules[f"pintlab.{name}"] = _Overlay(ours, theirs)
    config = importlib.import_module("pintlab.config")
    if "nccl" not in config.EXECUTORS:
        config.EXECUTORS = tuple(config.EXECUTORS) + ("nccl",)
    return importlib.import_module("pintlab.cli")


if __name__ == "__main__":
    sys.exit(install().main(sys.argv[1:]))
