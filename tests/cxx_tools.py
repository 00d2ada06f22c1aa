"""Build the C++ drop-in example (tests/cxx/iterate_example.cpp) against include/asdsm_b200.hpp
and the in-tree libasdsm_b200.so."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2303_01163_b200")


def build_example(tmpdir):
    exe = os.path.join(str(tmpdir), "iterate_example")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           "-o", exe, os.path.join(ROOT, "tests", "cxx", "iterate_example.cpp"), "-L", LIBDIR, "-lasdsm_b200",
           f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def run_example(exe, *args):
    p = subprocess.run([exe, *[str(a) for a in args]], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout
