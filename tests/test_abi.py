"""CPU checks of the C-ABI boundary: the library loads, exports every symbol
include/ibm.h declares, the ctypes structs match the header, and host-side
configuration validation works (no compute calls; no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import ibm_inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ibm.h")


@pytest.fixture(scope="module")
def ibm():
    from paper_2402_17337_b200 import build as B
    B.build()
    import paper_2402_17337_b200.ibm as M
    M.lib()
    return M


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"IBM_API\s+(?:int|const char\s*\*)\s*(ibm_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("ibm_init", "ibm_set_body", "ibm_step", "ibm_get_fields", "ibm_forces"):
        assert must in names  # BASELINE.json north_star boundary


def test_library_exports_every_declared_symbol(ibm):
    lib = ibm.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert sorted(ibm.EXPORTS) == declared_functions()


def test_exports_only_the_abi():
    import subprocess
    from paper_2402_17337_b200 import LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    text = [l.split()[-1] for l in out.splitlines() if " T " in l]
    assert sorted(text) == declared_functions()


def test_library_is_sm100a():
    import subprocess
    from paper_2402_17337_b200 import LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header(ibm, tmp_path):
    """Compile a C probe against include/ibm.h; the ctypes mirrors must agree."""
    import subprocess
    probe = tmp_path / "probe.c"
    probe.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "ibm.h"\n'
                     'int main(){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(ibm_config),'
                     ' offsetof(ibm_config, loopback), offsetof(ibm_config, nccl_id),'
                     ' sizeof(ibm_step_stats), offsetof(ibm_step_stats, status), offsetof(ibm_step_stats, ms), offsetof(ibm_step_stats, launches));'
                     'return 0;}\n')
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert vals == [C.sizeof(ibm.ibm_config), ibm.ibm_config.loopback.offset, ibm.ibm_config.nccl_id.offset,
                    C.sizeof(ibm.ibm_step_stats), ibm.ibm_step_stats.status.offset,
                    ibm.ibm_step_stats.ms.offset, ibm.ibm_step_stats.launches.offset]


def test_workspace_size_scales(ibm):
    small = I.cfg1()
    cfg = ibm.make_config(small.xn, small.yn, **small.solver_kwargs())
    n1 = ibm.ibm_workspace_size(cfg)
    big = I.cfg1(nx=256, ny=192)
    n2 = ibm.ibm_workspace_size(ibm.make_config(big.xn, big.yn, **big.solver_kwargs()))
    assert n1 > 0 and 3.0 < n2 / n1 < 4.5
    # ~19 fp64 arrays + 4 uint8 arrays per node
    assert n1 > 19 * 8 * 128 * 96


@pytest.mark.parametrize("field,value", [("nx", 3), ("Re", -1.0), ("dt", 0.0), ("omega_p", 2.0),
                                         ("omega_uv", 0.5), ("tol_p", 0.0), ("maxit_p", 0)])
def test_config_validation(ibm, field, value):
    c = I.cfg1()
    kw = c.solver_kwargs()
    xn, yn = c.xn, c.yn
    if field == "nx":
        xn = xn[:4]
    else:
        kw[field] = value
    cfg = ibm.make_config(xn, yn, **kw)
    with pytest.raises(ibm.IBMError) as e:
        ibm.ibm_workspace_size(cfg)
    assert e.value.status == ibm.IBM_ERR_CONFIG


def test_config_nonmonotone_axis(ibm):
    c = I.cfg1()
    xn = c.xn.copy()
    xn[5] = xn[4]
    with pytest.raises(ibm.IBMError):
        ibm.ibm_workspace_size(ibm.make_config(xn, c.yn, **c.solver_kwargs()))


def test_slab_rows_cover_grid(ibm):
    """Host slab partition: ny rows split into near-equal contiguous slabs."""
    c = I.cfg1()
    for P in (1, 2, 3, 4, 8):
        cfg = ibm.make_config(c.xn, c.yn, nranks=P, rank=0, loopback=True, **c.solver_kwargs())
        assert ibm.ibm_workspace_size(cfg) > 0
    # too many slabs for 96 rows (fewer than 4 rows each)
    with pytest.raises(ibm.IBMError):
        ibm.ibm_workspace_size(ibm.make_config(c.xn, c.yn, nranks=32, loopback=True, **c.solver_kwargs()))


def test_product_package_does_not_import_oracle():
    """The product path never routes through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2402_17337_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                src = open(os.path.join(root, f)).read()
                for bad in (r"\bimport\s+oracle", r"\bfrom\s+oracle", r"ibm_oracle", r"\borc_\w+\(",
                            r"libibm_oracle"):
                    assert not re.search(bad, src), (f, bad)
