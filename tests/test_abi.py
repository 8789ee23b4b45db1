"""The C-ABI library loads without a GPU and exports every declared symbol."""

import ctypes
import re

import numpy as np

from conftest import ROOT
from paper_2310_17739_b200 import _native as N


def declared_functions():
    text = (ROOT / "include" / "nucsim_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void)\s+(nsb_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "nsb_fuse" in names and "nsb_plan_run_mma" in names
    assert len(names) >= 25


def test_library_exports_every_declared_symbol():
    handle = ctypes.CDLL(str(N.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(handle, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared_functions()) == set(N.EXPORTS)
    N.lib()  # signatures apply cleanly


def test_op_record_layout_matches_header():
    assert N.OP_DTYPE.itemsize == 64
    assert N.OP_DTYPE.fields["mask"][1] == 56


def test_device_count_without_gpu_is_clean():
    assert N.device_count() >= 0


def test_status_codes_map_to_reference_exceptions():
    from paper_2310_17739_b200 import FilterAssertionError, ProjectionError, ResourceLimitError
    st = N.Status()
    st.step, st.prob = 4, 1e-15
    for code, exc in ((N.NSB_EINVAL, ValueError), (N.NSB_EASSERT, FilterAssertionError),
                      (N.NSB_EPROJECT, ProjectionError), (N.NSB_ERESOURCE, ResourceLimitError),
                      (N.NSB_EDEVICE, RuntimeError)):
        try:
            N.check(code, st)
        except exc as e:
            if code == N.NSB_EASSERT:
                assert e.step == 4 and e.prob == 1e-15
        else:
            raise AssertionError(code)


def test_gate_matrix_rejects_bad_tags():
    out = np.zeros(64, np.float64)
    assert N.lib().nsb_gate_matrix(999, None, 0, N.ptr(out)) == N.NSB_EINVAL
    assert N.lib().nsb_gate_matrix(0, None, 0, N.ptr(out)) == N.NSB_EINVAL  # u3 needs 3 params


def test_class_names_match_header():
    """nsb_plan_analyze writes NSB_N_CLASSES counts into the caller's buffer."""
    from paper_2310_17739_b200.workloads import CLASS_NAMES
    text = (ROOT / "include" / "nucsim_b200.h").read_text()
    n = int(re.search(r"#define NSB_N_CLASSES (\d+)", text).group(1))
    assert len(CLASS_NAMES) == n
