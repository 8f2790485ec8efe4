"""Build libzpir_b200.so in-tree for sm_100a (nvcc, no torch extension machinery).

    python -m paper_2603_09190_b200.build [--verbose]

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libzpir_b200.so")
SOURCES = ["capi.cu", "gemv.cu", "hint_gemm.cu", "answer.cu", "multiexp.cu", "umma_gemm.cu",
           "probe.cu", "chacha.cu", "conv.cu", "db_handle.cu", "tc_pippenger.cu", "compat.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    inc = os.path.join(HERE, "..", "include")
    deps += [os.path.join(inc, f) for f in os.listdir(inc)]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def conv_path():
    import sysconfig
    return os.path.join(HERE, "_zpir_conv" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_conv(force=False):
    """CPython extension for int <-> limb conversion at the API boundary."""
    import sysconfig
    out = conv_path()
    src = os.path.join(CSRC, "pyconv.c")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    tmp = out + ".tmp"
    subprocess.check_call(["gcc", "-O3", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"],
                           src, "-o", tmp])
    os.replace(tmp, out)
    return out


def build(verbose=False, force=False):
    build_conv(force)
    if not force and not needs_build():
        return LIB
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = os.path.join(HERE, "build", src.replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", os.path.join(HERE, "..", "include"), "-c", os.path.join(CSRC, src),
               "-o", obj, *os.environ.get("ZPIR_NVCC_EXTRA", "").split()]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
    tmp = LIB + ".tmp"
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True))
