"""CPU-side checks: the C-ABI library loads and exports every entry point of
include/pintlab_b200.h; host-side setup (quadrature, validation) matches the
reference.  No kernel is launched here (no GPU in the build container)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1407_6486_b200 import _build, _capi, hierarchy, multigrid as mg, quadrature
from paper_1407_6486_b200.heat import Grid, HeatOperator

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "pintlab_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(pl_\w+)\s*\(", src,
                                 re.M)))


def test_library_builds_and_exports_header():
    _build.build()
    lib = ctypes.CDLL(_build.LIB)
    decl = header_functions()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert set(decl) == set(_capi.EXPORTED)
    assert _capi.lib().pl_abi_version() == 1


def test_kind_names_and_stats_without_gpu():
    _capi.stats_reset()
    st = _capi.stats()
    assert "jacobi" in st and all(v == (0, 0.0) for v in st.values())


def test_bad_arguments_map_to_value_error():
    # argument validation happens before any device work
    rc = _capi.lib().pl_heat_apply(None, None, 4, 16, 1.0, 1.0, 2, None)
    assert rc == _capi.PL_ERR_ARG
    with pytest.raises(ValueError):
        _capi.check(rc)
    assert "bad grid" in _capi.last_error()


@pytest.mark.parametrize("m", range(1, 9))
def test_quadrature_matches_golden_tables(m):
    from oracle.pintlab_oracle import uniform_table, correction_interp, uniform_nodes
    t = quadrature.uniform_table(m)
    assert np.array_equal(t.q, uniform_table(m).q)
    for mc in range(1, m + 1):
        if m % mc == 0:
            p = quadrature.correction_interpolation(quadrature.uniform_nodes(mc),
                                                    quadrature.uniform_nodes(m))
            assert np.array_equal(p, correction_interp(uniform_nodes(mc), uniform_nodes(m)))


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        mg.MgConfig(smoother="sor")
    with pytest.raises(ValueError):
        mg.MgConfig(pre_sweeps=-1)
    with pytest.raises(ValueError):
        mg.FixedCycles(0)
    with pytest.raises(ValueError):
        mg.ToTolerance(tol=0.0)
    with pytest.raises(ValueError):
        mg.ToTolerance(stall=1.5)
    with pytest.raises(ValueError):
        Grid(4, 8)
    with pytest.raises(ValueError):
        Grid(1, 12)
    with pytest.raises(ValueError):
        HeatOperator(Grid(1, 8), 1.0, 3)
    with pytest.raises(ValueError):
        quadrature.uniform_nodes(0)


def test_hierarchy_checks():
    def lvl(n, m, order=2):
        return hierarchy.Level(HeatOperator(Grid(1, n), 1.0, order), quadrature.uniform_table(m),
                               mg.MgConfig(), mg.FixedCycles(1))
    hierarchy.check_hierarchy([lvl(32, 4), lvl(16, 2)])
    hierarchy.check_hierarchy([lvl(32, 4), lvl(32, 2)])
    with pytest.raises(ValueError):
        hierarchy.check_hierarchy([lvl(32, 4), lvl(8, 2)])
    with pytest.raises(ValueError):
        hierarchy.check_hierarchy([lvl(32, 2), lvl(16, 4)])
    with pytest.raises(ValueError):
        hierarchy.check_hierarchy([lvl(32, 4, 2), lvl(16, 2, 4)])
    with pytest.raises(ValueError):
        hierarchy.check_hierarchy([lvl(32, 4), lvl(16, 3)])
    with pytest.raises(ValueError):
        hierarchy.check_hierarchy([])
    with pytest.raises(ValueError):
        hierarchy.Level(HeatOperator(Grid(1, 8)), quadrature.uniform_table(2), mg.MgConfig(),
                        mg.FixedCycles(1), space_interp_order=3)


def test_seeded_field_recipe_matches_oracle():
    from oracle.pintlab_oracle import seeded_field
    from paper_1407_6486_b200.heat import seeded_field as product_field
    for d, n in ((1, 64), (2, 32), (3, 16)):
        assert np.array_equal(product_field(Grid(d, n)), seeded_field(d, n))


def test_policies_accepted_and_unknown_rejected():
    """Direct is on the GPU path now (pl_mg_direct); anything that is not a
    reference policy is a ValueError, never a silent substitute."""
    for pol in (mg.Direct(), mg.FixedCycles(1), mg.ToTolerance()):
        mg._check_policy(pol)
    with pytest.raises(ValueError):
        mg._check_policy("direct")


def test_comm_entry_points_validate_and_create_ids():
    """pl_comm_*: NCCL is opened lazily (the library loads without it); ids are
    128 bytes; argument errors are rejected before any device work."""
    import ctypes as C
    lib = _capi.lib()
    buf = C.create_string_buffer(128)
    assert lib.pl_comm_unique_id(buf) == 0
    assert any(buf.raw)
    assert lib.pl_comm_unique_id(None) < 0
    h = C.c_void_p()
    assert lib.pl_comm_init(C.byref(h), buf, 2, 1, 0) < 0          # rank >= nranks
    assert lib.pl_comm_init(C.byref(h), buf, 0, 0, 0) < 0          # no ranks
    assert lib.pl_comm_send(None, None, 0, 0, None) < 0
    assert lib.pl_comm_recv(None, None, 0, 0, None) < 0
    assert lib.pl_comm_bcast(None, None, 0, 0, None) < 0
    assert lib.pl_comm_destroy(None) == 0
