"""In-tree build of libmagiplan.so (host C++20 planner + sm_100a CUDA kernels).

Every translation unit is compiled by nvcc for ``sm_100a`` only, with
``-lineinfo`` so ncu source pages map back to the kernels, and linked into one
shared library exporting the C ABI declared in ``include/magiplan.h``. The
library travels to GPU boxes inside the repo snapshot (it is git-ignored, not
gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
# diagnostics build (python -m paper_2505_13211_b200.build --trace): the
# per-role event tracer of the FFA kernels (tools/trace_*.py) is compiled in
# only with -DMAGI_TRACE; the default library carries one instantiation per
# kernel and head_dim
TRACE = "--trace" in sys.argv
LIB = PKG / "libmagiplan.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [
    "-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
    f"-I{ROOT / 'include'}", f"-I{ROOT / 'third_party'}", f"-I{CSRC}",
]
CUDA_FLAGS = ["-Xptxas", "-v", "--expt-relaxed-constexpr"]
if TRACE:  # separate objects and library: never replaces the product build
    COMMON.append("-DMAGI_TRACE")
    OBJ = ROOT / "build" / "obj_trace"
    LIB = ROOT / "build" / "trace" / "libmagiplan.so"


def _sources() -> list[Path]:
    srcs = sorted((CSRC / "host").glob("*.cpp")) + sorted((CSRC / "kernels").glob("*.cu"))
    return srcs


def _headers_mtime() -> float:
    hdrs = [*CSRC.rglob("*.h"), *CSRC.rglob("*.hpp"), *CSRC.rglob("*.cuh"), *CSRC.rglob("*.inc")]
    hdrs += list((ROOT / "include").rglob("*.h"))
    return max((h.stat().st_mtime for h in hdrs), default=0.0)


def _compile(src: Path, hdr_mtime: float, verbose: bool) -> tuple[Path, str]:
    obj = OBJ / (src.parent.name + "_" + src.name + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return obj, ""
    cmd = ["nvcc", *ARCH, *COMMON]
    if src.suffix == ".cu":
        cmd += CUDA_FLAGS
    else:
        cmd += ["-x", "cu"] if False else []
    cmd += ["-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    log = res.stdout + res.stderr
    return obj, log


def build(verbose: bool = False) -> Path:
    srcs = _sources()
    hdr_mtime = _headers_mtime()
    newest = max([hdr_mtime] + [s.stat().st_mtime for s in srcs])
    if LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB  # up to date (e.g. the prebuilt library shipped to a GPU box)
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(lambda s: _compile(s, hdr_mtime, verbose), srcs))
    objs = [o for o, _ in results]
    logs = "".join(l for _, l in results)
    (ROOT / "build" / "ptxas.log").write_text(logs)
    if not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = ["nvcc", *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart_static"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(logs)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
