"""Builds libsphinx.so (all hot-path kernels + the C ABI) in-tree for sm_100a.

    python -m paper_2511_18672_b200.build        # or __graft_entry__.build()

nvcc cross-compiles on a CPU-only box; the .so travels to the GPU box with the repo.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libsphinx.so")
SOURCES = ["abi.cu", "block_mask.cu", "compact.cu", "noise_inject.cu", "sparse_conv3x3.cu",
           "scatter_cached.cu", "ddim_step.cu",
           "uncertainty_map.cu", "group_norm.cu", "temporal_attn.cu", "block_copy.cu", "shard_plan.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared",
              "-cudart", "static"]


def _stale():
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "sphinx.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, trace=False):
    """trace=True builds the dev-only variant libsphinx_trace.so (-DSPHINX_TRACE timelines and the
    -DSPHINX_DEV_KNOBS A/B environment knobs); the release libsphinx.so reads no environment
    variable except SPHINX_PDL."""
    so = SO.replace("libsphinx.so", "libsphinx_trace.so") if trace else SO
    if not trace and not force and not _stale():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
        (["-DSPHINX_TRACE", "-DSPHINX_DEV_KNOBS"] if trace else []) + \
        ["-I", os.path.join(ROOT, "include"), "-o", so + ".tmp"] + [os.path.join(CSRC, s) for s in SOURCES]
    subprocess.check_call(cmd)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    if "--trace" in sys.argv:
        print(build(trace=True))
        sys.exit(0)
    build(force=True, verbose="-v" in sys.argv)
    print(SO)
