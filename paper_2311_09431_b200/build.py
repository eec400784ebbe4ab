"""Build the in-tree CUDA library ``libstriped_attn.so`` for sm_100a with nvcc.

``python -m paper_2311_09431_b200.build`` (or ``__graft_entry__.build()``).  The .so is
git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libstriped_attn.so")
BUILD = os.path.join(PKG, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")] + os.environ.get("SA_NVCC_EXTRA", "").split()


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "striped_attn.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    out = out or OUT
    if not force and not _needs_build() and out == OUT:
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), sources()))
    tmp = out + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


PROBE_SRC = os.path.join(ROOT, "tests", "csrc", "probe.cu")
PROBE_OUT = os.path.join(ROOT, "tests", "csrc", "libsa_probe.so")


def build_probe(force: bool = False) -> str:
    """Test-only library (tcgen05 / TMA layout probes): tests/csrc/libsa_probe.so.  Kept
    out of the product library; shares only the header-only device helpers."""
    if not force and os.path.exists(PROBE_OUT) and \
            os.path.getmtime(PROBE_OUT) > max(os.path.getmtime(PROBE_SRC),
                                              os.path.getmtime(os.path.join(CSRC, "common.cuh"))):
        return PROBE_OUT
    tmp = PROBE_OUT + ".tmp"
    cmd = [NVCC, *ARCH, *FLAGS, "-I" + CSRC, "-shared", PROBE_SRC, "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for probe.cu:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, PROBE_OUT)
    return PROBE_OUT


if __name__ == "__main__":
    outs = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")]
    print(build(force="--force" in sys.argv or bool(outs), verbose="-v" in sys.argv,
                out=outs[0] if outs else None))
