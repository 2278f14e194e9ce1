"""The C++ drop-in surface (include/polycert_b200.hpp): the reference's
analyzer known-answer tests written against the same C++ names
(proj/tests/test_analyzer.cpp:44-122), compiled with g++ and linked against
the in-tree CUDA library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "build", "test_facade")
LIBDIR = os.path.join(ROOT, "paper_2007_10868_b200")


def _build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", LIBDIR, "-lpolycert_b200", f"-Wl,-rpath,{LIBDIR}", "-o", OUT],
                   check=True, capture_output=True, text=True)
    return OUT


def test_facade_compiles_and_links():
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_facade_known_answers():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "facade ok" in r.stdout
