"""Host-side checks of the C-ABI library (-m "not gpu"): it loads, exports every symbol
include/ifctn.h declares, and validates arguments before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def abi():
    from paper_2511_16358_b200 import build
    build.build()
    from paper_2511_16358_b200 import _abi
    return _abi


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ifctn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ifctn_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(abi):
    names = declared_functions()
    assert len(names) >= 15
    L = abi.lib()
    for n in names:
        assert hasattr(L, n), n
        assert n in abi.SIGNATURES, f"{n} missing from the Python binding"
    assert set(abi.SIGNATURES) == set(names)


def test_binding_flags_match_the_header(abi):
    """Every IFCTN_FLAG_* of include/ifctn.h has the same value in the binding (a drift would
    silently select another kernel path), and the flags are distinct bits."""
    src = open(os.path.join(ROOT, "include", "ifctn.h")).read()
    flags = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+(IFCTN_FLAG_[A-Z0-9_]+)\s+(\d+)u", src)}
    assert len(flags) >= 9 and flags["IFCTN_FLAG_NONE"] == 0
    for name, val in flags.items():
        assert getattr(abi, name) == val, name
    bits = [v for v in flags.values() if v]
    assert all(v & (v - 1) == 0 for v in bits) and len(set(bits)) == len(bits)


def test_library_is_sm100a(abi):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(abi):
    assert abi.ifctn_status_string(0) == "IFCTN_OK"
    assert abi.ifctn_status_string(3) == "IFCTN_E_RANKS"
    assert abi.ifctn_status_string(99) == "IFCTN_E_UNKNOWN"


def ranks_flat(N, R):
    r = np.full((N, N), R, dtype=np.int32)
    np.fill_diagonal(r, 0)
    return list(r.reshape(-1))


def test_workspace_bytes_validation(abi):
    ws = abi.ifctn_workspace_bytes(3, (256, 256, 31), ranks_flat(3, 4), abi.IFCTN_F32)
    assert ws > 256 * 256 * 31 * 4
    assert ws == abi.ifctn_workspace_bytes(3, (256, 256, 31), ranks_flat(3, 4), abi.IFCTN_F32)
    bad = ranks_flat(3, 4)
    bad[1] = 5  # R_{0,1} != R_{1,0}
    with pytest.raises(abi.IfctnError, match="E_RANKS"):
        abi.ifctn_workspace_bytes(3, (4, 4, 4), bad, abi.IFCTN_F32)
    bad = ranks_flat(3, 4)
    bad[0] = 1  # diagonal
    with pytest.raises(abi.IfctnError, match="E_RANKS"):
        abi.ifctn_workspace_bytes(3, (4, 4, 4), bad, abi.IFCTN_F32)
    with pytest.raises(abi.IfctnError, match="E_RANKS"):
        abi.ifctn_workspace_bytes(3, (4, 4, 4), ranks_flat(3, 0), abi.IFCTN_F32)
    with pytest.raises(abi.IfctnError, match="E_UNSUPPORTED"):
        abi.ifctn_workspace_bytes(3, (4, 4, 4), ranks_flat(3, 65), abi.IFCTN_F32)
    with pytest.raises(abi.IfctnError, match="E_SHAPE"):
        abi.ifctn_workspace_bytes(1, (4,), [0], abi.IFCTN_F32)
    with pytest.raises(abi.IfctnError, match="E_SHAPE"):
        abi.ifctn_workspace_bytes(7, (2,) * 7, ranks_flat(7, 1), abi.IFCTN_F32)
    with pytest.raises(abi.IfctnError, match="E_SHAPE"):
        abi.ifctn_workspace_bytes(3, (4, 0, 4), ranks_flat(3, 1), abi.IFCTN_F32)
    with pytest.raises(abi.IfctnError, match="E_ARG"):
        abi.ifctn_workspace_bytes(3, (4, 4, 4), ranks_flat(3, 1), 7)


def test_create_validates_before_device_work(abi):
    x = np.zeros(8, np.float32)
    m = np.ones(8, np.uint8)
    g = np.zeros(3 * 2 * 2 * 2, np.float32)
    P = lambda a: ctypes.c_void_p(a.ctypes.data)
    with pytest.raises(abi.IfctnError, match="E_ARG"):   # rho <= 0
        abi.ifctn_create(3, (2, 2, 2), ranks_flat(3, 2), abi.IFCTN_F32, 0.0, P(x), P(m), P(g),
                         None, 0, None, None, 0)
    with pytest.raises(abi.IfctnError, match="E_ARG"):   # NULL observed
        abi.ifctn_create(3, (2, 2, 2), ranks_flat(3, 2), abi.IFCTN_F32, 0.1, None, P(m), P(g),
                         None, 0, None, None, 0)
    with pytest.raises(abi.IfctnError, match="E_NO_OBSERVED"):
        abi.ifctn_create(3, (2, 2, 2), ranks_flat(3, 2), abi.IFCTN_F32, 0.1, P(x),
                         P(np.zeros(8, np.uint8)), P(g), None, 0, None, None, 0)


def test_shard_ranges(abi):
    """Reading R21: ⌈I/W⌉ slices first; shard mode = largest, the first on ties (SURVEY §8(e):
    C5 shards along mode 1 = API mode 0)."""
    dims = (214, 61, 144, 4)
    sizes = []
    for r in range(8):
        d = abi.ifctn_dist(None, r, 8, -1)
        sm, b, e = abi.ifctn_shard_range(4, dims, d)
        assert sm == 0
        sizes.append(e - b)
        if r:
            assert b == prev_e
        prev_e = e
    assert sizes == [27] * 6 + [26] * 2 and prev_e == 214
    d = abi.ifctn_dist(None, 1, 8, -1)
    assert abi.ifctn_shard_range(4, (144, 176, 3, 50), d) == (1, 22, 44)
    assert abi.ifctn_shard_range(3, (64, 64, 32), abi.ifctn_dist(None, 0, 2, -1))[0] == 0
    assert abi.ifctn_shard_range(3, (32, 64, 64), abi.ifctn_dist(None, 0, 2, -1))[0] == 1
    assert abi.ifctn_shard_range(5, (64, 64, 64, 64, 32), abi.ifctn_dist(None, 0, 8, -1)) == (0, 0, 8)
    assert abi.ifctn_shard_range(3, (8, 8, 8), None) == (0, 0, 8)


def test_python_package_has_no_fallback():
    src = open(os.path.join(ROOT, "paper_2511_16358_b200", "__init__.py")).read()
    src += open(os.path.join(ROOT, "paper_2511_16358_b200", "_abi.py")).read()
    assert "oracle" not in src.replace("TEST INFRASTRUCTURE", "")
    for f in os.listdir(os.path.join(ROOT, "paper_2511_16358_b200")):
        if f.endswith(".py"):
            assert "import oracle" not in open(os.path.join(ROOT, "paper_2511_16358_b200", f)).read()


def test_header_is_plain_c(tmp_path):
    """include/ifctn.h is a C-ABI header: it compiles as C99 (no C++ or CUDA types) and a C
    program can link against libifctn.so with it."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "use.c"
    src.write_text('#include "include/ifctn.h"\n#include <stdio.h>\n'
                   'int main(void) {\n'
                   '  int64_t dims[3] = {4, 5, 6}; int32_t r[9] = {0,2,2, 2,0,2, 2,2,0}; size_t b = 0;\n'
                   '  ifctn_status s = ifctn_workspace_bytes(3, dims, r, IFCTN_F32, NULL, &b);\n'
                   '  printf("%s %zu\\n", ifctn_status_string(s), b);\n'
                   '  return s == IFCTN_OK && b > 0 ? 0 : 1;\n}\n')
    lib = os.path.join(root, "paper_2511_16358_b200")
    exe = tmp_path / "use"
    subprocess.check_call([gcc, "-std=c99", "-Wall", "-Werror", "-I", root, str(src), "-o", str(exe),
                           "-L", lib, "-lifctn", f"-Wl,-rpath,{lib}"])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("IFCTN_OK")


def test_binding_validates_buffers_before_the_call(abi):
    """The binding checks dtype, element count (local shard / factor layout) and contiguity
    of every buffer before its raw address crosses the ABI — a float64 G⁰ for a float32
    problem, a view, or a buffer of the wrong extent raises E_ARG instead of being read as
    garbage (all rejected before any device work, so this runs without a GPU)."""
    from paper_2511_16358_b200 import IfctnError, Solver, num_params
    dims, R = (6, 5, 4), 2
    n = int(np.prod(dims))
    obs = np.zeros(n, np.float32)
    mask = np.ones(n, np.uint8)
    g0 = np.zeros(num_params(dims, R), np.float32)
    cases = [
        (obs.astype(np.float64), mask, g0, "dtype"),                # O of another dtype than G⁰
        (obs, mask, g0.astype(np.float64), "dtype"),                # G⁰ float64, O float32
        (obs[:-1], mask, g0, "elements"),                           # short O
        (obs, mask[:-3], g0, "elements"),                           # short mask
        (obs, mask, g0[:-1], "elements"),                           # short G⁰
        (np.zeros(2 * n, np.float32)[::2], mask, g0, "contiguous"),  # strided view
        (obs, mask.astype(np.int32), g0, "dtype"),                  # mask not bytes
    ]
    for o, m, g, what in cases:
        with pytest.raises(IfctnError, match=f"E_ARG.*{what}"):
            Solver(dims, R, o, m, g)
    with pytest.raises(IfctnError, match="E_ARG.*dtype"):
        Solver(dims, R, obs, mask, g0, dtype=abi.IFCTN_F64)        # declared dtype wins
