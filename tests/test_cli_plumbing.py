"""The reference's own CLI (pintlab.cli) on this package's hot path: the
plumbing of tools/pintlab_cli_gpu.py, on CPU.

The launcher overlays this package's modules on the reference's names for
the accelerated path and hands argv to the reference's ``cli.main``;
configuration parsing, presets, validation, CSV and footer stay the
reference's code.  Needs the reference package (present in the build
container only; skipped elsewhere).  Without a GPU the product path must
refuse to run (no CPU fallback), after the reference's parsing and
validation have accepted the configuration.
"""
import os
import sys

import pytest

REF = "/root/reference/pkg/src"
if not os.path.isdir(REF):
    pytest.skip("reference package not present (GPU box)", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cli():
    saved = {k: v for k, v in sys.modules.items() if k == "pintlab" or k.startswith("pintlab.")}
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import pintlab_cli_gpu
    mod = pintlab_cli_gpu.install()
    yield mod
    for k in [k for k in sys.modules if k == "pintlab" or k.startswith("pintlab.")]:
        del sys.modules[k]
    sys.modules.update(saved)
    sys.path.remove(REF)


def test_accelerated_names_resolve_to_this_package(cli):
    from paper_1407_6486_b200 import heat, hierarchy, multigrid, pfasst, sdc
    assert cli.pfasst_run is pfasst.pfasst_run
    assert cli.run_sdc is sdc.run_sdc
    assert cli.Level is hierarchy.Level
    assert cli.HeatOperator is heat.HeatOperator
    assert cli.MgConfig is multigrid.MgConfig
    # off-path helpers stay the reference's own (exact solutions for the CSV)
    assert cli.exact_pde.__module__ == "pintlab.heat"


def test_config_validation_is_the_references(cli, capsys):
    assert cli.main(["single-run", "--set", "executor=mpi"]) == 2
    assert "executor must be one of" in capsys.readouterr().err
    assert cli.main(["single-run", "--set", "nodes=notanumber"]) == 2


def test_nccl_executor_and_presets_build_device_levels(cli):
    from paper_1407_6486_b200 import hierarchy
    cfg = cli.parse_config(None, {"executor": "nccl"}, **dict(cli.PRESETS["strong-3d"],
                                                               experiment="strong-3d"))
    cfg = cli.validate_sub(cfg)
    assert cfg.executor == "nccl"
    levels = cli.build_levels(cfg)
    assert all(isinstance(lv, hierarchy.Level) for lv in levels)
    assert [lv.operator.order for lv in levels][0] == cfg.orders[0]
    assert levels[0].mg_cfg.smoother == "jor-rb"


def test_product_path_fails_loudly_without_a_gpu(cli, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    out = tmp_path / "run.csv"
    with pytest.raises(RuntimeError, match="CUDA device"):
        cli.main(["single-run", "--set", "variant=IPFASST", "--set", "levels=2",
                  "--set", "nodes=3,2", "--set", "orders=2,2", "--set", "policy=fixed:1",
                  "--set", "n_x=32", "--set", "n_t=4", "--set", "p=4",
                  "--set", "executor=nccl", "--set", f"out={out}"])
