"""The C++ drop-in adapter (include/parbfs_gpu.hpp) compiles against the
UNMODIFIED reference headers and links with the reference library plus
libpbfs.so; run here (no GPU) it must surface the C ABI's device error as a
parbfs::Error (no CPU fallback), and on a GPU box with the reference present
it runs the reference's own time_run over gpu::kernel_fn()."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/core/include"
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libparbfs_ref.so")
LIB = os.path.join(ROOT, "paper_2503_00430_b200")

PROGRAM = r"""
#include <cstdio>
#include <cstring>
#include "parbfs/generator.hpp"
#include "parbfs/graph_stats.hpp"
#include "parbfs/timing.hpp"
#include "parbfs_gpu.hpp"
int main() {
  using namespace parbfs;
  const CsrGraph g = generate({GeneratorKind::Kronecker, 12, 16, 3});
  KernelConfig cfg;
  cfg.variant = KernelVariant::Hybrid;
  try {
    // the reference's own oracle-checked timer driving the GPU through the plugin slot
    const TimingReport rep = time_run(g, 0, cfg, 3, 1, gpu::kernel_fn());
    std::printf("GPU %lld\n", static_cast<long long>(rep.median.count()));
    return 0;
  } catch (const Error& e) {
    std::printf("ERROR %s\n", e.what());
    return std::strstr(e.what(), "no CUDA device") ? 3 : 1;
  }
}
"""


@pytest.mark.skipif(not (os.path.isdir(REF_INC) and os.path.exists(REF_SO)),
                    reason="needs the reference headers and oracle/_ref")
def test_adapter_compiles_against_reference_and_has_no_cpu_fallback(tmp_path):
    src = tmp_path / "adapter.cpp"
    src.write_text(PROGRAM)
    exe = tmp_path / "adapter"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
                    str(src), REF_SO, os.path.join(LIB, "libpbfs.so"),
                    f"-Wl,-rpath,{os.path.dirname(REF_SO)}:{LIB}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    try:
        import torch
        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    if gpu:
        assert r.returncode == 0 and r.stdout.startswith("GPU"), r.stdout + r.stderr
    else:
        assert r.returncode == 3, r.stdout + r.stderr


ADAPTER = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["criterion1", "timerun", "multi"])
def test_reference_drives_the_b200_through_the_cpp_adapter(mode):
    # tests/cpp/adapter_check.cpp, prebuilt here against the unmodified
    # reference headers (make -C oracle adapter) and shipped with the repo:
    # acceptance criterion 1 through gpu::run_bfs (200 graphs, each rebuilt in
    # the same stack slot), the reference's own oracle-checked time_run over
    # gpu::kernel_fn(), equal-sized graphs at one address, and the
    # LevelObserver.
    assert os.path.exists(ADAPTER), "oracle/_ref/adapter_check must travel with the repo"
    r = subprocess.run([ADAPTER, mode], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.startswith(("OK", "time_run")), r.stdout + r.stderr
    assert "OK" in r.stdout
