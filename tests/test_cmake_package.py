"""The CMake package: a downstream project written for the reference's exported target
(find_package(kernelweave) + kernelweave::core) configures, builds and runs its host logic."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(shutil.which("cmake") is None, reason="cmake not on PATH")
def test_downstream_project_builds(tmp_path):
    (tmp_path / "CMakeLists.txt").write_text(
        "cmake_minimum_required(VERSION 3.20)\nproject(app CXX)\nfind_package(kernelweave REQUIRED)\n"
        "add_executable(app main.cpp)\ntarget_link_libraries(app PRIVATE kernelweave::core)\n")
    (tmp_path / "main.cpp").write_text(
        "#include <kernelweave/kernelweave.hpp>\n#include <cstdio>\nusing namespace kernelweave;\n"
        "int main() {\n"
        "  const WorkDiv wd = kernels::axpyWorkDiv(BackendKind::GpuCudaRt, 1 << 20, 512, 4);\n"
        "  std::printf(\"%zu\\n\", totalExtent(wd, Level::Grid, Unit::Elems)[0]);\n"
        "  return wd.blocksPerGrid()[0] == 512 ? 0 : 1;\n}\n")
    b = tmp_path / "build"
    cfg = subprocess.run(["cmake", "-S", str(tmp_path), "-B", str(b), f"-Dkernelweave_DIR={ROOT / 'cmake'}"],
                         capture_output=True, text=True, timeout=300)
    assert cfg.returncode == 0, cfg.stdout + cfg.stderr
    bld = subprocess.run(["cmake", "--build", str(b)], capture_output=True, text=True, timeout=300)
    assert bld.returncode == 0, bld.stdout + bld.stderr
    run = subprocess.run([str(b / "app")], capture_output=True, text=True, timeout=60)
    assert run.returncode == 0 and run.stdout.strip() == str(1 << 20)
