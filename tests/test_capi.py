"""The drop-in boundary: libpbfs.so loads on a CPU-only host, exports every
entry point include/pbfs.h declares, and its structs have the layout the C
header gives them (checked by compiling the header with gcc)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2503_00430_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pbfs.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pbfs_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(L.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    bound = {name for name, _, _ in L.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_struct_layout_matches_header(tmp_path):
    structs = {"pbfs_csr": L.Csr, "pbfs_config": L.Config, "pbfs_level": L.Level,
               "pbfs_run_info": L.RunInfo, "pbfs_graph_options": L.GraphOptions,
               "pbfs_graph_info": L.GraphInfo, "pbfs_gen_spec": L.GenSpec,
               "pbfs_stats": L.Stats}
    src = tmp_path / "sz.c"
    body = "".join(f'printf("{k} %zu\\n", sizeof({k}));' for k in structs)
    src.write_text(f'#include <stdio.h>\n#include "pbfs.h"\nint main(void){{{body}return 0;}}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    sizes = {k: int(v) for k, v in (line.split() for line in out.splitlines())}
    for k, cls in structs.items():
        assert sizes[k] == ctypes.sizeof(cls), k


def test_abi_version_and_status_strings():
    assert L.lib.pbfs_abi_version() == 2
    assert L.lib.pbfs_status_string(0) == b"ok"
    assert L.lib.pbfs_status_string(4) == b"capacity error"


def test_config_defaults_match_reference():
    # kernel_config.hpp:38-70
    c = L.Config()
    L.lib.pbfs_config_init(ctypes.byref(c))
    assert (c.variant, c.worker_count, c.hybrid_threshold_fraction, c.alpha, c.beta,
            c.flush_capacity) == (1, 1, 0.05, 15.0, 18.0, 4096)
    assert L.lib.pbfs_config_validate(ctypes.byref(c)) == 0
    c.hybrid_threshold_fraction = 0.0
    assert L.lib.pbfs_config_validate(ctypes.byref(c)) == 2


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device error path")
def test_no_cpu_fallback_without_device():
    import paper_2503_00430_b200 as pb
    from graphs import make_path
    g = make_path(8)
    with pytest.raises(pb.Error, match="no CUDA device"):
        pb.run_bfs(g, 0, pb.KernelConfig(variant=pb.KernelVariant.Hybrid), pb.compute_stats(g))
