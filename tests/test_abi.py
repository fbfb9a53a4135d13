"""CPU: the C-ABI library loads and exports every symbol include/se2map.h declares (no compute calls)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "se2map.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(se2m_[a-z_0-9]+)\s*\(", src)))


def test_library_builds_loads_and_exports():
    from paper_2503_02412_b200 import _build
    lib_path = _build.build()
    lib = ctypes.CDLL(lib_path)
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    from paper_2503_02412_b200 import se2map
    assert sorted(se2map.EXPORTS) == names


def test_params_struct_layout_matches_header():
    """The ctypes mirror of se2m_params has the header's size (checked against the C compiler)."""
    import subprocess
    import tempfile
    from paper_2503_02412_b200 import se2map
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "s.c")
        open(c, "w").write('#include "se2map.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                           'int main(){printf("%zu %zu %zu\\n", sizeof(se2m_params), '
                           'offsetof(se2m_params, robot_x), offsetof(se2m_params, cuda_stream));return 0;}\n')
        exe = os.path.join(d, "s")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c])
        size, off_rx, off_st = map(int, subprocess.check_output([exe]).split())
    assert ctypes.sizeof(se2map.Params) == size
    assert se2map.Params.robot_x.offset == off_rx
    assert se2map.Params.cuda_stream.offset == off_st


def test_default_params_without_gpu():
    from paper_2503_02412_b200 import se2map
    p = se2map.default_params()
    assert (p.nx, p.ny, p.n_yaw) == (100, 100, 36)
    assert abs(p.phi_x_max - 0.52) < 1e-15 and abs(p.kappa_max - 0.1) < 1e-15
    assert list(p.w_r) == [0.4, 0.3, 0.3]


def test_no_oracle_import_in_product():
    """The product package never imports the oracle (parity independence)."""
    pkg = os.path.join(ROOT, "paper_2503_02412_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "se2_oracle" not in s, f
