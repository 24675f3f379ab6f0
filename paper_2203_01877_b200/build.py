"""Build libtqp.so in-tree with nvcc for sm_100a (B200). No torch extension, no JIT cache."""

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libtqp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(ROOT, "include", "tqp.h"), __file__]


STAMP = LIB + ".flags"


def _flag_stamp():
    """The nvcc flags a build uses, TQP_NVCC_EXTRA included: an A/B build with extra flags
    (tools/ab_*.sh) must not be mistaken for the default one."""
    return " ".join(FLAGS + os.environ.get("TQP_NVCC_EXTRA", "").split())


def needs_build():
    if not os.path.exists(LIB):
        return True
    try:
        with open(STAMP) as f:
            if f.read() != _flag_stamp():
                return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force=False, verbose=False, jobs=None):
    if not force and not needs_build():
        return LIB
    objs = []
    procs = []
    odir = os.path.join(PKG, "build")
    os.makedirs(odir, exist_ok=True)
    for s in sources():
        o = os.path.join(odir, os.path.basename(s) + ".o")
        # TQP_NVCC_EXTRA: extra nvcc flags for A/B experiments (e.g. "-DTQP_PEER_MATCH_ANY=0")
        cmd = [NVCC, *FLAGS, *os.environ.get("TQP_NVCC_EXTRA", "").split(), "-c", s, "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(o)
    failed = []
    for s, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        if p.returncode != 0:
            failed.append(s)
    if failed:
        raise RuntimeError("nvcc failed for: " + ", ".join(failed))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
                           "-lcudart"])
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(_flag_stamp())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
