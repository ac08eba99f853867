"""Compile examples/c_abi_demo.c against the in-tree libpfsched.so with plain gcc (no torch)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "c_abi_demo.c")
EXE = os.path.join(HERE, "c_abi_demo")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build() -> str:
    libdir = os.path.join(ROOT, "paper_2507_10150_b200")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", SRC, "-I", os.path.join(ROOT, "include"),
                           "-I", os.path.join(CUDA, "include"), "-L", libdir, "-lpfsched",
                           "-L", os.path.join(CUDA, "lib64"), "-lcudart",
                           "-Wl,-rpath," + libdir, "-Wl,-rpath," + os.path.join(CUDA, "lib64"), "-o", EXE])
    return EXE


if __name__ == "__main__":
    print(build())
