"""Bounds-checked runs (compute-sanitizer is not available on the GPU pool).

    python tools/checked_runs.py build      # here: tools/libmmas_checked.so (-DMMAS_CHECKED)
    python tools/checked_runs.py [pytest args]   # on the GPU: the parity tests of the paths with
                                                 # device checks (MMAS_CHECK in kernels.cuh /
                                                 # construct.cuh) against that library

A failed check traps the kernel (the test then fails with a CUDA launch error); every test
still compares its results with the oracle."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "tools", "libmmas_checked.so")
TESTS = ["tests/test_fallback_compact_gpu.py", "tests/test_parity_gpu.py", "tests/test_parity_full_gpu.py",
         "tests/test_lean_gpu.py", "tests/test_colonies_gpu.py"]


def main():
    if sys.argv[1:2] == ["build"]:
        from paper_2003_11902_b200 import build as b
        cmd = [b.NVCC, *b.NVCC_FLAGS, "-DMMAS_CHECKED", "-I", os.path.join(ROOT, "include"), "-o", SO, *b.SOURCES]
        subprocess.run(cmd, check=True, capture_output=True)
        print(SO)
        return
    env = dict(os.environ, MMAS_LIB=SO)
    args = sys.argv[1:] or ["-x", "-q"]
    sys.exit(subprocess.run([sys.executable, "-m", "pytest", "-m", "gpu", *args, *TESTS], env=env, cwd=ROOT).returncode)


if __name__ == "__main__":
    main()
