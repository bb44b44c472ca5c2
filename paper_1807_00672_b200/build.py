"""In-tree build of the native library and the test-only oracle.

    python -m paper_1807_00672_b200.build        # or __graft_entry__.build()

Products (git-ignored, travel to the GPU box with the snapshot):
  paper_1807_00672_b200/libswe_b200.so   CUDA kernels (sm_100a) + C-ABI
                                         (include/swe_dev.h, include/swe_host.h)
  tests/cpp/api_driver                   C++ drop-in API driver (include/swe/*.hpp)
  oracle/liboracle.so, oracle/_ref/libswe_ref.so   test-only checkers
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INC = ROOT / "include"
BUILD = PKG / "_build"
LIB = PKG / "libswe_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: the reference is built with -ffp-contract=off
# (CMakeLists.txt:17-18); no contraction keeps every FP64 op bit-identical.
NVFLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", f"-I{INC}", f"-I{CSRC}"]
CXXFLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-fvisibility=hidden",
            f"-I{INC}", "-I/usr/local/cuda/include"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def build_library(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(INC.glob("*.h")) + list((INC / "swe").glob("*.hpp"))
    cu = CSRC / "swe_dev.cu"
    cu_o = BUILD / "swe_dev.o"
    host = CSRC / "host_abi.cpp"
    host_o = BUILD / "host_abi.o"
    if force or _stale(cu_o, [cu, *headers]):
        _run([NVCC, *ARCH, *NVFLAGS, "-c", cu, "-o", cu_o], verbose)
    if force or _stale(host_o, [host, *headers]):
        _run(["g++", *CXXFLAGS, "-c", host, "-o", host_o], verbose)
    if force or _stale(LIB, [cu_o, host_o]):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, cu_o, host_o], verbose)
    return LIB


def build_api_driver(verbose: bool = False, force: bool = False) -> Path:
    src = ROOT / "tests" / "cpp" / "api_driver.cpp"
    out = ROOT / "tests" / "cpp" / "api_driver"
    if not src.exists():
        return out
    headers = list((INC / "swe").glob("*.hpp")) + list(INC.glob("*.h"))
    if force or _stale(out, [src, LIB, *headers]):
        _run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", f"-I{INC}", src, "-o", out,
              f"-L{PKG}", "-lswe_b200", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../../paper_1807_00672_b200"],
             verbose)
    return out


def build_multigpu_driver(verbose: bool = False, force: bool = False) -> Path:
    """tests/cpp/multigpu_driver.cpp: the multi-GPU path of the drop-in API
    (include/swe/multigpu.hpp) driven as a reference caller would."""
    src = ROOT / "tests" / "cpp" / "multigpu_driver.cpp"
    out = ROOT / "tests" / "cpp" / "multigpu_driver"
    headers = list((INC / "swe").glob("*.hpp")) + list(INC.glob("*.h"))
    if force or _stale(out, [src, LIB, *headers]):
        _run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", f"-I{INC}", src, "-o", out,
              f"-L{PKG}", "-lswe_b200", "-pthread",
              "-Wl,-rpath,$ORIGIN/../../paper_1807_00672_b200"], verbose)
    return out


JSON_INC = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/"
                "thirdparty/nlohmann")
REF_INC = Path("/root/reference/proj/include")


def build_harness_driver(verbose: bool = False, force: bool = False) -> Path:
    """The reference's own bench/convergence harness (its bench.hpp, included
    in place) compiled against this repo's drop-in headers -- only where the
    reference exists; the binary travels to the GPU box prebuilt."""
    src = ROOT / "tests" / "cpp" / "harness_driver.cpp"
    out = ROOT / "tests" / "cpp" / "harness_driver"
    if not (REF_INC.exists() and (JSON_INC / "json.hpp").exists()):
        return out
    headers = list((INC / "swe").glob("*.hpp")) + list(INC.glob("*.h"))
    if force or _stale(out, [src, LIB, *headers]):
        _run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", f"-I{INC}", f"-I{REF_INC}",
              f"-I{JSON_INC}", src, "-o", out, f"-L{PKG}", "-lswe_b200",
              "-Wl,-rpath,$ORIGIN/../../paper_1807_00672_b200"], verbose)
    return out


REF_TESTS = Path("/root/reference/proj/tests")
REF_UNIT_SOURCES = ["test_kernels", "test_engine", "test_mesh", "test_cases", "test_io",
                    "test_harness", "doctest_main"]


def _build_doctest_binary(out: Path, sources, include_dirs, link, verbose, force, extra=()):
    """Compile the reference's own doctest sources (read in place, not copied)
    with the doctest stand-in tests/cpp/doctest/doctest.h, one object per
    source, in parallel."""
    shim = ROOT / "tests" / "cpp" / "doctest" / "doctest.h"
    deps = [shim, *[REF_TESTS / f"{n}.cpp" for n in sources]]
    if link and LIB.exists():
        deps += [LIB, *(INC / "swe").glob("*.hpp")]
    if not force and not _stale(out, deps):
        return out
    obj_dir = BUILD / ("objs_" + out.name)
    obj_dir.mkdir(parents=True, exist_ok=True)
    flags = ["-std=c++20", "-O2", "-ffp-contract=off", f"-I{shim.parent}",
             *[f"-I{d}" for d in include_dirs], f"-I{JSON_INC}", f"-I{REF_TESTS}", *extra]
    procs, objs = [], []
    for n in sources:
        o = obj_dir / f"{n}.o"
        objs.append(o)
        cmd = ["g++", *flags, "-c", REF_TESTS / f"{n}.cpp", "-o", o]
        if verbose:
            print(" ".join(str(c) for c in cmd), flush=True)
        procs.append(subprocess.Popen([str(c) for c in cmd]))
    if any(p.wait() for p in procs):
        raise subprocess.CalledProcessError(1, f"compile {out.name}")
    out.parent.mkdir(parents=True, exist_ok=True)
    _run(["g++", *extra, *objs, "-o", out, *link], verbose)
    return out


def build_reference_tests(verbose: bool = False, force: bool = False) -> None:
    """The reference's own unit tests (test_kernels/engine/mesh/cases/io/
    harness.cpp) and acceptance suite compiled UNCHANGED against the drop-in
    headers (include/ first on the path, so swe/engine.hpp etc. are this
    repo's; the reference's io.hpp / bench.hpp come from its tree) ->
    tests/cpp/ref_unit, tests/cpp/ref_acceptance (every engine call on the
    B200); and against the reference alone -> oracle/_ref/ref_unit_cpu, which
    checks the doctest stand-in itself.  Only where /root/reference exists;
    the binaries travel to the GPU box prebuilt."""
    if not (REF_TESTS.exists() and (JSON_INC / "json.hpp").exists()):
        return
    link = [f"-L{PKG}", "-lswe_b200", "-Wl,-rpath,$ORIGIN/../../paper_1807_00672_b200"]
    # acceptance.cpp's criterion 10 drives the CLI tool (needs CLI11, absent):
    # the path is a stub and the test is excluded at run time
    cli = ['-DSWE_CLI_PATH="/bin/false"']
    _build_doctest_binary(ROOT / "tests" / "cpp" / "ref_unit", REF_UNIT_SOURCES,
                          [INC, REF_INC], link, verbose, force)
    _build_doctest_binary(ROOT / "tests" / "cpp" / "ref_acceptance", ["acceptance"],
                          [INC, REF_INC], link, verbose, force, extra=cli)
    _build_doctest_binary(ROOT / "oracle" / "_ref" / "ref_unit_cpu", REF_UNIT_SOURCES,
                          [REF_INC], [], verbose, force, extra=["-fopenmp"])


def build_io_ext_driver(verbose: bool = False, force: bool = False) -> Path:
    """tests/cpp/io_ext_driver.cpp: the parallel VTK writer and backend.gpus
    next to the reference's io.hpp (needs /root/reference + json.hpp; the
    binary travels prebuilt)."""
    src = ROOT / "tests" / "cpp" / "io_ext_driver.cpp"
    out = ROOT / "tests" / "cpp" / "io_ext_driver"
    if not (REF_INC.exists() and (JSON_INC / "json.hpp").exists()):
        return out
    headers = list((INC / "swe").glob("*.hpp")) + list(INC.glob("*.h"))
    if force or _stale(out, [src, LIB, *headers]):
        _run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", f"-I{INC}", f"-I{REF_INC}",
              f"-I{JSON_INC}", src, "-o", out, f"-L{PKG}", "-lswe_b200", "-pthread",
              "-Wl,-rpath,$ORIGIN/../../paper_1807_00672_b200"], verbose)
    return out


def build_oracle(verbose: bool = False) -> None:
    _run(["make", "-s", "-C", ROOT / "oracle"], verbose)


def build_all(verbose: bool = False, force: bool = False) -> None:
    build_library(verbose, force)
    build_api_driver(verbose, force)
    build_multigpu_driver(verbose, force)
    build_harness_driver(verbose, force)
    build_io_ext_driver(verbose, force)
    build_oracle(verbose)
    build_reference_tests(verbose, force)


if __name__ == "__main__":
    build_all(verbose=True, force="--force" in sys.argv)
