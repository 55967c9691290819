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


def header_prototypes():
    """{name: (return type, [parameter types])} of every function declared in
    include/pintlab_b200.h (comments stripped, prototypes may span lines)."""
    src = open(os.path.join(ROOT, "include", "pintlab_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", " ", src, flags=re.S)
    src = re.sub(r"^\s*#.*$", " ", src, flags=re.M)
    out = {}
    for m in re.finditer(r"((?:const\s+)?[A-Za-z_][\w ]*?[\s*]+)(pl_\w+)\s*\(([^)]*)\)\s*;",
                         src, re.S):
        ret, name, params = m.group(1), m.group(2), m.group(3)
        ret = " ".join(ret.replace("*", " * ").split())
        plist = []
        for prm in params.split(","):
            prm = " ".join(prm.replace("*", " * ").split())
            if prm in ("", "void"):
                continue
            # drop the parameter name (the last identifier) when one is given
            toks = prm.split()
            if len(toks) > 1 and re.fullmatch(r"[A-Za-z_]\w*", toks[-1]) and \
                    toks[-1] not in ("int", "double", "char", "void", "size_t", "unsigned",
                                     "long"):
                toks = toks[:-1]
            plist.append(" ".join(toks))
        out[name] = (ret, plist)
    return out


def header_functions():
    return sorted(header_prototypes())


def _ctypes_kind(t):
    """The ctypes type a C type must be bound with (pointers -> void* or a
    typed pointer; width matters for integers and floats)."""
    t = t.replace("const ", "")
    if t.endswith("*"):
        return "ptr"
    return {"int": ctypes.c_int, "unsigned": ctypes.c_uint, "double": ctypes.c_double,
            "size_t": ctypes.c_size_t, "long long": ctypes.c_longlong}[t]


def _bound_kind(ct):
    if ct in (ctypes.c_void_p, ctypes.c_char_p) or (isinstance(ct, type) and
                                                    issubclass(ct, ctypes._Pointer)):
        return "ptr"
    return ct


def test_library_builds_and_exports_header():
    _build.build()
    lib = ctypes.CDLL(_build.LIB)
    decl = header_functions()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert set(decl) == set(_capi.EXPORTED)
    assert _capi.lib().pl_abi_version() == 2


def test_ctypes_signatures_match_header_prototypes():
    """Arity and argument widths of every binding equal the C prototype: a
    missing argument would let ctypes truncate a trailing 64-bit stream
    handle to a C int."""
    protos = header_prototypes()
    for name, (ret, params) in protos.items():
        res, args = _capi._SIGS[name]
        assert len(args) == len(params), (name, params, args)
        for i, (c_t, bound) in enumerate(zip(params, args)):
            assert _ctypes_kind(c_t) == _bound_kind(bound), (name, i, c_t, bound)
        want = None if ret == "void" else _ctypes_kind(ret)
        assert want == _bound_kind(res), (name, ret, res)


def test_header_parser_sees_multiline_and_long_long():
    protos = header_prototypes()
    assert protos["pl_field_elems"] == ("long long", ["int", "int"])
    assert len(protos["pl_sdc_sweep"][1]) == 16
    assert protos["pl_sdc_residual"][1][7:9] == ["int", "int"]
    assert protos["pl_last_error"] == ("const char *", [])


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
