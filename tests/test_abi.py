"""The C-ABI boundary (include/kz_b200.h): the library loads without a GPU
and exports every declared symbol; status codes map onto the reference's
exception taxonomy (errors.py)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "kz_b200.h")).read()
    return sorted(set(re.findall(r"^KZ_API\s+[\w\s\*]+?\b(kz_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_binding_list():
    from paper_2401_17474_b200 import _native as N

    assert header_functions() == sorted(N.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    import ctypes

    from paper_2401_17474_b200 import _native as N

    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert N.load_library().kz_version() >= 1


def test_no_device_is_reported_not_crashed():
    from paper_2401_17474_b200 import _native as N

    n = N.device_count()
    assert n >= 0
    if n == 0:
        from paper_2401_17474_b200 import DeviceSystem

        with pytest.raises(N.NativeUnavailable):
            DeviceSystem(m=4, n=2)


def test_status_mapping():
    from paper_2401_17474_b200 import _native as N
    from paper_2401_17474_b200.errors import DegenerateRowError, EmptyRangeError

    N.check(N.KZ_OK)
    with pytest.raises(DegenerateRowError) as ei:
        N.check(N.KZ_EDEGENERATE, bad_row=7)
    assert ei.value.row == 7
    with pytest.raises(EmptyRangeError):
        N.check(N.KZ_EEMPTYRANGE)
    with pytest.raises(ValueError):
        N.check(N.KZ_EINVAL)
    with pytest.raises(MemoryError):
        N.check(N.KZ_ENOMEM)
    with pytest.raises(N.NativeError):
        N.check(N.KZ_ECUDA)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2401_17474_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text and "kzo_" not in text, f


def _header_struct_fields(name):
    """Field names of a typedef'd struct in include/kz_b200.h, in order."""
    src = open(os.path.join(ROOT, "include", "kz_b200.h")).read()
    m = re.search(r"typedef struct\s*\{([^{}]*)\}\s*" + name + r"\s*;", src)
    assert m, name
    body = re.sub(r"/\*.*?\*/", "", m.group(1), flags=re.S)
    return re.findall(r"\b(\w+)\s*;", body)


def test_ctypes_structs_match_the_header():
    """The ctypes mirrors of kz_params / kz_result (the package's _native and the stub a maintainer
    copies from INTEGRATION.md) list the header's fields in order: kz_solve writes every field of
    kz_result, so a shorter mirror would be written past."""
    from paper_2401_17474_b200 import _native as N

    for name, cls in (("kz_params", N.Params), ("kz_result", N.Result)):
        assert [f[0] for f in cls._fields_] == _header_struct_fields(name), name
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    for name, cls in (("kz_params", "_Params"), ("kz_result", "_Result")):
        m = re.search(r"class " + cls + r"\(C\.Structure\):.*?_fields_ = \[(.*?)\]\n", doc, flags=re.S)
        assert m, cls
        assert re.findall(r'\("(\w+)"', m.group(1)) == _header_struct_fields(name), name
