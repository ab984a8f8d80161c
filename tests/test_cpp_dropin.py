"""The reference-facing C++ API: a program written against the reference's
headers (tests/cpp/dropin_test.cpp) builds and links against the B200
library.  CPU: compile + host plan checks.  GPU: the training checks."""
import os
import pathlib
import shutil
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "dropin_test.cpp"
BIN = ROOT / "tests" / "cpp" / "dropin_test"
LIB = ROOT / "paper_2410_14312_b200" / "lib"


def _build():
    if BIN.exists() and BIN.stat().st_mtime >= SRC.stat().st_mtime and \
            BIN.stat().st_mtime >= (LIB / "libpipesim_b200.so").stat().st_mtime:
        return
    cxx = shutil.which("g++") or "g++"
    subprocess.run([cxx, "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(SRC),
                    f"-L{LIB}", "-lpipesim_b200", f"-Wl,-rpath,{LIB}", "-o", str(BIN)],
                   check=True)


def test_dropin_compiles_and_plan_checks_pass():
    _build()
    r = subprocess.run([str(BIN), "--plan-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "all checks passed" in r.stdout


@pytest.mark.gpu
def test_dropin_training_on_gpu():
    _build()
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "all checks passed" in r.stdout
