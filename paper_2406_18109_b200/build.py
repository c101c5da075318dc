"""Build ``libdk_b200.so`` in-tree with nvcc for sm_100a (no GPU needed)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdk_b200.so")
SOURCES = ["dk_runtime.cu", "dk_kernels.cu", "dk_jit.cu", "dk_comm.cu", "dk_pcg.cu"]
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _nccl_dirs() -> tuple[str, str]:
    import nvidia.nccl  # torch's bundled NCCL (2.28.x), the one torch.distributed loads

    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc_cmd() -> list[str]:
    inc, lib = _nccl_dirs()
    return [
        os.path.join(CUDA, "bin", "nvcc"),
        "-gencode",
        "arch=compute_100a,code=sm_100a",
        "-O3",
        "-lineinfo",
        "-std=c++17",
        "-shared",
        "-Xcompiler",
        "-fPIC",
        "-Xptxas",
        "-v",
        f"-I{inc}",
        f"-I{os.path.join(HERE, '..', 'include')}",
        *[os.path.join(CSRC, s) for s in SOURCES],
        "-o",
        LIB,
        f"-L{os.path.join(CUDA, 'lib64', 'stubs')}",
        f"-L{os.path.join(CUDA, 'lib64')}",
        f"-L{lib}",
        "-lcuda",
        "-lnvrtc",
        "-l:libnccl.so.2",
        f"-Xlinker=-rpath,{lib}",
        f"-Xlinker=-rpath,{os.path.join(CUDA, 'lib64')}",
    ]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "dk_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = nvcc_cmd()
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(HERE, "csrc", "build.log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed (see {log})")
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
