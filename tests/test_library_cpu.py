"""CPU-side checks of the C-ABI library (no compute calls: there is no GPU here)."""
import ctypes
import os
import subprocess

import pytest

import paper_2006_06775_b200 as bdm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(bdm.LIB_PATH):
        subprocess.check_call(["make", "-s", "paper_2006_06775_b200/libbdm.so"], cwd=ROOT)
    return bdm.load_library()


def test_header_symbols_exported(lib):
    names = bdm.header_symbols()
    assert {"bdm_init", "bdm_grid_build", "bdm_mech_step", "bdm_get_displacements"} <= set(names)
    for name in names:
        assert hasattr(lib, name), name
    # the binding wraps every declared symbol under the same name
    assert set(names) == set(bdm._SIGS)


def test_defaults_and_errors_without_gpu(lib):
    p = bdm.bdm_params_default()
    assert (p.k_rep, p.gamma_att, p.adherence, p.dt, p.eta, p.max_disp, p.box_edge_min) == (
        10.0, 4.0, 0.1, 1.0, 1.0, 3.0, 0.0)
    assert lib.bdm_abi_version() == 1
    h = ctypes.c_void_p()
    # argument validation happens before any device call
    assert lib.bdm_init(ctypes.byref(h), -1, None, None, ctypes.byref(p)) == bdm.BDM_EINVAL
    assert b"n = -1" in lib.bdm_last_error(None)
    bad = bdm.bdm_params_default(eta=0.0)
    assert lib.bdm_init(ctypes.byref(h), 0, None, None, ctypes.byref(bad)) == bdm.BDM_EINVAL
    assert lib.bdm_mech_step(None, 1) == bdm.BDM_EINVAL
    lib.bdm_destroy(None)


def test_sass_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", bdm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", bdm.LIB_PATH], capture_output=True, text=True).stdout
    assert "DADD" in sass and "DMUL" in sass and "k_force" in sass


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2006_06775_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "bdm_oracle" not in txt, f
