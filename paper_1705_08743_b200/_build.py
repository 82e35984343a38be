"""Build the sm_100a C-ABI library in-tree: paper_1705_08743_b200/libsemimat_b200.so.

nvcc cross-compiles for sm_100a without a GPU, so this runs in the build
container; the .so is git-ignored but travels to the GPU box with the repo
snapshot.  Objects are compiled in parallel.  The library is rebuilt when the
content hash of its inputs (every source and header, the nvcc flags and the
nvcc version) differs from the one recorded beside it at the last build
(libsemimat_b200.so.stamp), not on file times: a fresh checkout or a copied
tree with newer mtimes but the same sources does not rebuild, and an edited
source with an older mtime does.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_obj"
LIB = PKG / "libsemimat_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                     "--expt-relaxed-constexpr", f"-I{REPO / 'include'}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the semimat_b200 CUDA library cannot be built")


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _deps():
    return _sources() + sorted(CSRC.glob("*.cuh")) + sorted((REPO / "include").glob("*.h"))


STAMP = LIB.with_name(LIB.name + ".stamp")


def _input_hash() -> str:
    import hashlib
    h = hashlib.sha256()
    for p in _deps():
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS + os.environ.get("SMX_EXTRA_NVCC_FLAGS", "").split()).encode())
    try:
        h.update(subprocess.run([_nvcc(), "--version"], capture_output=True, text=True).stdout.encode())
    except (RuntimeError, OSError):
        pass
    return h.hexdigest()


def up_to_date() -> bool:
    if not LIB.exists() or not STAMP.exists():
        return False
    return STAMP.read_text().strip() == _input_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    nvcc = _nvcc()
    OBJ.mkdir(exist_ok=True)

    def compile_one(src: Path) -> Path:
        obj = OBJ / (src.stem + ".o")
        # SMX_EXTRA_NVCC_FLAGS: tuning experiments only (e.g. -DSMX_PACKED_BK=32)
        extra = os.environ.get("SMX_EXTRA_NVCC_FLAGS", "").split()
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "--cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    STAMP.write_text(_input_hash() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
