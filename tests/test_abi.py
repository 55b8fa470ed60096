"""CPU checks of the boundary: libmrrr_b200.so loads without a GPU and exports
every function include/mrrr.h declares; the Python binding's names match."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mrrr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:int|void|size_t|char)\s*\*?\s*(mrrr_\w+)\s*\(", src, re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def so():
    from paper_1205_2107_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = header_functions()
    for required in ["mrrr_stemr", "mrrr_stemr_dist", "mrrr_stemr_nccl", "mrrr_stemr_host", "mrrr_workspace_bytes",
                     "mrrr_strerror", "mrrr_default_opts", "mrrr_get_stats", "mrrr_version"]:
        assert required in names


def test_library_exports_every_symbol(so):
    lib = ctypes.CDLL(so)
    for name in header_functions():
        assert hasattr(lib, name), name


def test_host_only_calls(so):
    from paper_1205_2107_b200 import mrrr as M
    L = M.lib()
    assert L.mrrr_strerror(0) == b"success"
    assert L.mrrr_strerror(-3) == b"invalid argument"
    assert L.mrrr_strerror(2).startswith(b"child")
    assert L.mrrr_workspace_bytes(20000, 20000) > 20000 * 20000 * 8 // 32
    o = M.default_opts()
    assert o.tol_relgap == 1e-3 and o.rtol_class == 2.0 ** -20 and o.max_depth == 128
    assert o.perturb_root == 1
    assert M.version().startswith("mrrr-b200")
    st = M.last_stats()
    assert set(st) >= {"nodes", "ms_k_vectors", "vec_elems"}


def test_nccl_entry_rejects_null_communicator(so):
    """mrrr_stemr_nccl validates its communicator before touching NCCL or CUDA."""
    from paper_1205_2107_b200 import mrrr as M
    rc = M.lib().mrrr_stemr_nccl(4, None, None, 0, 0.0, 0.0, 0, 0, None, None, None, None, None, None, None, 4, None)
    assert rc == -9


def test_load_sets_work_queues_unless_set(so):
    """include/mrrr.h "Process environment": loading the library sets
    CUDA_DEVICE_MAX_CONNECTIONS=32 only when the caller has not set it."""
    import subprocess
    import sys
    code = ("import ctypes, sys; ctypes.CDLL(sys.argv[1]); g = ctypes.CDLL(None).getenv; "
            "g.restype = ctypes.c_char_p; print(g(b'CUDA_DEVICE_MAX_CONNECTIONS').decode())")
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    out = subprocess.run([sys.executable, "-c", code, so], env=env, capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "32"
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "8"
    out = subprocess.run([sys.executable, "-c", code, so], env=env, capture_output=True, text=True, check=True)
    assert out.stdout.strip() == "8"


def test_stats_struct_matches_header():
    """The ctypes Stats/Opts layouts mirror mrrr_stats_t / mrrr_opts_t."""
    from paper_1205_2107_b200 import mrrr as M
    src = open(os.path.join(ROOT, "include", "mrrr.h")).read()
    body = re.search(r"typedef struct \{((?:(?!typedef).)*?)\} mrrr_stats_t;", src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"(\w+);", body)
    assert fields == [f for f, _ in M.Stats._fields_]
    body = re.search(r"typedef struct \{((?:(?!typedef).)*?)\} mrrr_opts_t;", src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    assert re.findall(r"(\w+);", body) == [f for f, _ in M.Opts._fields_]


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1205_2107_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "mrrr_oracle" not in txt, f
