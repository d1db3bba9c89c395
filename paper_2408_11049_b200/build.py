"""Build the sm_100a shared libraries in-tree with nvcc (no JIT cache, no torch extension).

  paper_2408_11049_b200/libmagicdec_b200.so   the product: csrc/*.cu behind include/magicdec_b200.h
  paper_2408_11049_b200/libmagicdec_b200_debug.so  the same with -DMD_DEBUG: device-side
                                              preconditions trap (tests/test_gpu_debug.py)
  synth/libmd_synth.so                        the GPU twin of the seeded input generators

Run `python -m paper_2408_11049_b200.build` (or __graft_entry__.build()).  Rebuilds only
when a source is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-cudart", "static", "--expt-relaxed-constexpr", "-Xptxas", "-v"]

LIB = os.path.join(HERE, "libmagicdec_b200.so")
DEBUG_LIB = os.path.join(HERE, "libmagicdec_b200_debug.so")
SYNTH_LIB = os.path.join(ROOT, "synth", "libmd_synth.so")


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _nvcc(sources, out, extra=(), log=None, force=False):
    deps = list(sources) + glob.glob(os.path.join(os.path.dirname(sources[0]), "*.cuh")) + \
        glob.glob(os.path.join(os.path.dirname(sources[0]), "*.h")) + [os.path.join(ROOT, "include", "magicdec_b200.h")]
    if not force and not _stale(out, deps):
        return False
    # one nvcc per translation unit, in parallel, then one link (the units share no device code)
    from concurrent.futures import ThreadPoolExecutor
    objs = [out + "." + os.path.splitext(os.path.basename(s))[0] + ".o" for s in sources]
    compile_flags = [f for f in FLAGS if f not in ("-shared", "-cudart", "static")]
    cmds = [[NVCC, *ARCH, *compile_flags, *extra, "-c", "-o", o, s] for s, o in zip(sources, objs)]
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC", "-o", out + ".tmp", *objs]
    if all(r.returncode == 0 for r in results):
        results.append(subprocess.run(link, capture_output=True, text=True))
    if log is not None:
        with open(log, "w") as f:
            for c, r in zip(cmds + [link], results):
                f.write(" ".join(c) + "\n" + r.stdout + r.stderr)
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    bad = [r for r in results if r.returncode != 0]
    if bad:
        sys.stderr.write("".join(r.stdout + r.stderr for r in bad))
        raise RuntimeError(f"nvcc failed building {out}")
    os.replace(out + ".tmp", out)
    return True


def build(force: bool = False, verbose: bool = False) -> None:
    srcs = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
    # export only the md_* C ABI: default-visibility for the extern "C" entry points
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=2) as ex:
        dbg = ex.submit(_nvcc, srcs, DEBUG_LIB, extra=["-DMD_BUILD", "-DMD_DEBUG"], force=force)
        built = _nvcc(srcs, LIB, extra=["-DMD_BUILD"], log=os.path.join(HERE, "build_ptxas.log"), force=force)
        dbuilt = dbg.result()
    sbuilt = _nvcc([os.path.join(ROOT, "synth", "csrc", "synth_gen.cu")], SYNTH_LIB, force=force)
    if verbose:
        print(f"libmagicdec_b200.so: {'built' if built else 'up to date'}; "
              f"libmagicdec_b200_debug.so: {'built' if dbuilt else 'up to date'}; "
              f"libmd_synth.so: {'built' if sbuilt else 'up to date'}")


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
