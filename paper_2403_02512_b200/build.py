"""Build libsvb200.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_2403_02512_b200.build [--force]

Sources: paper_2403_02512_b200/csrc/*.cu|*.cpp -> paper_2403_02512_b200/libsvb200.so,
linked against the NCCL that ships with torch (nvidia-nccl-cu12, 2.28.x) via rpath so only
one libnccl.so.2 is ever loaded into a process.
"""

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsvb200.so")
BUILD = os.path.join(HERE, "..", "build", "svb200")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl-cu12 (torch's NCCL) not found")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def cuda_home():
    return os.path.dirname(os.path.dirname(os.path.realpath(nvcc())))


def gen_dev_inc():
    """fused_dev.cuh as a C++ raw string: the device helpers the runtime pass compiler (fused_jit.cpp,
    NVRTC) prepends to every generated pass kernel -- the same source the prebuilt kernel includes."""
    with open(os.path.join(CSRC, "fused_dev.cuh")) as f:
        body = f.read()
    text = 'R"SVB200DEV(' + body + ')SVB200DEV"\n'
    out = os.path.join(BUILD, "fused_dev_src.inc")
    if not os.path.exists(out) or open(out).read() != text:
        with open(out, "w") as f:
            f.write(text)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "svb200.h")]
    return any(os.path.getmtime(s) > t for s in deps)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    inc, lib = nccl_dirs()
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", inc, "-I", os.path.join(HERE, "..", "include"),
              "-I", BUILD]
    gen_dev_inc()
    cmds = []
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(HERE, "..", "include", "svb200.h")]
    t_hdr = max(os.path.getmtime(x) for x in hdrs)
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        # incremental: an object newer than its source and every header is reused
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), t_hdr):
            continue
        cmd = [nvcc(), *ARCH, "-lineinfo", *common, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
            cmd += ["--expt-relaxed-constexpr"]
        else:
            cmd = [nvcc(), *common, "-I", os.path.join(cuda_home(), "include"), "-x", "c++", "-c", src, "-o", obj]
        cmds.append((src, cmd))
    # compile the translation units in parallel (fused.cu alone takes ~2 min)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds) or 1, os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda sc: (sc[0], subprocess.run(sc[1], capture_output=True, text=True)), cmds))
    for src, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
    tmp = OUT + ".tmp"
    link = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-L", lib, "-l:libnccl.so.2",
            "-Xlinker", "-rpath", "-Xlinker", lib, "-cudart", "static",
            "-L", os.path.join(cuda_home(), "lib64"), "-lnvrtc", "-Xlinker", "-rpath", "-Xlinker", os.path.join(cuda_home(), "lib64")]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
