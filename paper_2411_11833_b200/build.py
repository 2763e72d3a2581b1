"""Build libtamp.so in-tree with nvcc for sm_100a (B200).  No JIT cache: the .so travels with the repo."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# one translation unit per instantiation group so the (slow) k_particle variants compile in parallel
SRCS = [os.path.join(HERE, "csrc", f) for f in ("tamp_api.cu", "tamp_kernels.cu", "tamp_particle_hinge.cu",
                                                 "tamp_particle_smooth.cu", "tamp_particle_serial.cu",
                                                 "tamp_particle_hinge_rich.cu", "tamp_particle_hinge_wide.cu", "tamp_particle_hinge_16.cu")]
HDRS = [os.path.join(HERE, "csrc", "tamp_program.h"), os.path.join(HERE, "csrc", "particle.cuh"),
        os.path.join(HERE, "csrc", "particle_serial.cuh"), os.path.join(HERE, "csrc", "particle_launch.cuh"),
        os.path.join(ROOT, "include", "tamp.h")]
LIB = os.path.join(HERE, "libtamp.so")
OBJ_DIR = os.path.join(HERE, "csrc", "build")
# the particle kernels use the approximate (MUFU-based, ~1-2 ulp) fp32 division and square root: no slow-path
# branches in the step loop; the parity tolerances (1e-4 relative cost) are orders of magnitude wider
FAST_DIV_SQRT = ["-prec-div=false", "-prec-sqrt=false"]
FAST_UNITS = ("tamp_particle_hinge.cu", "tamp_particle_smooth.cu", "tamp_particle_serial.cu", "tamp_kernels.cu",
              "tamp_particle_hinge_rich.cu", "tamp_particle_hinge_wide.cu", "tamp_particle_hinge_16.cu")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in SRCS + HDRS)


def build(force=False, verbose=False):
    """Compile csrc/*.cu into paper_2411_11833_b200/libtamp.so (sm_100a).  Returns the path.

    Serialised by an exclusive file lock: concurrent callers (one process per GPU under torchrun, pytest
    workers) wait for the first one's build instead of writing the same objects."""
    if not force and up_to_date():
        return LIB
    import fcntl
    os.makedirs(OBJ_DIR, exist_ok=True)
    with open(os.path.join(OBJ_DIR, ".lock"), "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        try:
            if not force and up_to_date():     # built by another process while we waited
                return LIB
            return _build(verbose)
        finally:
            fcntl.flock(lock, fcntl.LOCK_UN)


def build_variant(name, defines, verbose=False, flags=()):
    """A/B build of the same sources with extra -D defines (and nvcc flags) into exp/<name>/libtamp.so (in-tree,
    git-ignored; bench --lib loads it).  Not part of the product build."""
    out = os.path.join(ROOT, "exp", name)
    return _build(verbose, defines=defines, obj_dir=os.path.join(out, "obj"), lib=os.path.join(out, "libtamp.so"),
                  flags=flags)


def _build(verbose=False, defines=(), obj_dir=OBJ_DIR, lib=LIB, flags=()):
    os.makedirs(obj_dir, exist_ok=True)
    objs = [os.path.join(obj_dir, os.path.basename(s)[:-3] + ".o") for s in SRCS]
    procs = [subprocess.Popen([nvcc()] + NVCC_FLAGS + (FAST_DIV_SQRT if os.path.basename(s) in FAST_UNITS else [])
                              + [f"-D{d}" for d in defines] + list(flags) + ["-c", "-o", o, s], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for s, o in zip(SRCS, objs)]
    logs, failed = [], []
    for s, p in zip(SRCS, procs):
        out, err = p.communicate()
        logs.append(f"== {os.path.basename(s)}\n{out}{err}")
        if p.returncode != 0:
            failed.append(s)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(logs))
    res = subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib + ".tmp"]
                         + objs, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    os.replace(lib + ".tmp", lib)
    with open(os.path.join(os.path.dirname(lib), "ptxas_info.txt"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
