"""Build the CUDA engine in-tree: csrc/*.cu -> _lib/libbinpaths_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a (B200 only), -lineinfo for ncu
source mapping, static cudart so the .so travels to the GPU box alone.
Run: python -m paper_1701_03512_b200.build
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_lib", "libbinpaths_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "static",
         "--expt-relaxed-constexpr", "-diag-suppress", "177"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh")) +
                              glob.glob(os.path.join(HERE, "csrc", "*.h")) +
                              [os.path.join(HERE, "..", "include", "binpaths_b200.h")])


def _stale_units(force: bool = False) -> list:
    """Units whose object is missing or older than its source or any header."""
    headers = [d for d in deps() if not d.endswith(".cu")]
    newest_header = max(os.path.getmtime(h) for h in headers)
    return [u for u in units() if force or not os.path.exists(u[2]) or
            os.path.getmtime(u[2]) < max(newest_header, os.path.getmtime(u[0]))]


def up_to_date() -> bool:
    """Per object, not per library: a library linked from objects compiled
    before a later source edit is stale even if it is newer than the edit."""
    if not os.path.exists(OUT) or _stale_units():
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(u[2]) <= t for u in units())


def fast_parts() -> int:
    import re
    with open(os.path.join(HERE, "csrc", "bp_kernels.h")) as f:
        return int(re.search(r"kFastParts = (\d+)", f.read()).group(1))


def units():
    """(source, extra nvcc flags, object) per translation unit; the K1
    instantiation file is compiled once per part."""
    out = []
    for src in sources():
        base = os.path.join(HERE, "_lib", "obj", os.path.basename(src)[:-3])
        if src.endswith("bp_exact_fast_inst.cu"):
            out += [(src, [f"-DBP_FAST_PART={i}"], f"{base}_{i}.o") for i in range(fast_parts())]
        else:
            out.append((src, [], base + ".o"))
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    """One nvcc per translation unit, in parallel (the template-heavy kernel
    files dominate), then one host link with static cudart."""
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.join(HERE, "_lib", "obj"), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    compile_flags = [f for f in FLAGS if f != "-shared"]
    from concurrent.futures import ThreadPoolExecutor

    def run(u):
        src, extra, obj = u
        cmd = [nvcc, *ARCH, *compile_flags, *extra, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        return subprocess.call(cmd)

    # incremental: an object is rebuilt when its source or any header is newer
    all_units = units()
    todo = _stale_units(force)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        rcs = list(ex.map(run, todo))
    failed = [u[0] + " " + " ".join(u[1]) for u, rc in zip(todo, rcs) if rc != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {failed}")
    tmp = OUT + ".tmp"
    subprocess.check_call([nvcc, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC",
                           "-o", tmp, *[u[2] for u in all_units]])
    os.replace(tmp, OUT)
    return OUT


def build_example() -> str:
    """examples/bp_price.c: a plain C client of the C ABI (header + .so only)."""
    root = os.path.dirname(HERE)
    src = os.path.join(root, "examples", "bp_price.c")
    out = os.path.join(root, "examples", "bp_price")
    lib = build()
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(src), os.path.getmtime(lib)):
        return out
    subprocess.check_call([os.environ.get("CC", "cc"), "-O2", "-std=c11", "-Wall", "-I", os.path.join(root, "include"),
                           src, "-o", out, "-L", os.path.dirname(lib), "-lbinpaths_b200",
                           "-Wl,-rpath,$ORIGIN/../paper_1701_03512_b200/_lib", "-lm"])
    return out


def build_variant(name: str, defines, parts=None, all_units: bool = False, sources=None) -> str:
    """Diagnostics: the library with extra -D flags on the K1 instantiation
    parts (all parts, or the listed ones) and on the units of the listed
    source basenames (sources=[...]); every unit with all_units=True
    -> _lib/variants/<name>.so, for
    BINPATHS_LIB=... scans (tools/scan_variants.sh).  Other objects are
    shared with the main build."""
    build()
    nvcc = os.environ.get("NVCC", "nvcc")
    compile_flags = [f for f in FLAGS if f != "-shared"]
    vdir = os.path.join(HERE, "_lib", "variants", name)
    os.makedirs(vdir, exist_ok=True)
    objs, procs = [], []
    for src, extra, obj in units():
        part = next((int(e.split("=")[1]) for e in extra if e.startswith("-DBP_FAST_PART=")), None)
        if part is not None:
            chosen = all_units or parts is None or part in parts
        else:
            chosen = all_units or (sources is not None and os.path.basename(src) in sources)
        if not chosen:
            objs.append(obj)
            continue
        vobj = os.path.join(vdir, os.path.basename(obj))
        objs.append(vobj)
        procs.append(subprocess.Popen([nvcc, *ARCH, *compile_flags, *extra, *[f"-D{d}" for d in defines],
                                       "-c", "-o", vobj, src]))
    if any(p.wait() != 0 for p in procs):
        raise subprocess.CalledProcessError(1, f"variant {name}")
    out = os.path.join(HERE, "_lib", "variants", name + ".so")
    subprocess.check_call([nvcc, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC", "-o", out, *objs])
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
