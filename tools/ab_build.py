#!/usr/bin/env python
"""Build an A/B pair of the native library for same-box comparisons:
exp/libA.so (+ exp/libA_prof.so) from git revision REV and exp/libB.so
(+ exp/libB_prof.so) from the working tree.  Run either with
AA_LIB_PATH=exp/libX.so (tools/knob_sweep.py) or tools/fa_prof.py --lib.

    python tools/ab_build.py HEAD
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXP = os.path.join(ROOT, "exp")


def build_tree(tree, tag, extra_flags=()):
    pkg = os.path.join(tree, "paper_2505_23520_b200")
    csrc = os.path.join(pkg, "csrc")
    nvcc = "/usr/local/cuda/bin/nvcc"
    arch = ["-gencode", "arch=compute_100a,code=sm_100a"]
    flags = arch + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                    "-I", os.path.join(tree, "include"), "-I", csrc]
    cus = sorted(f for f in os.listdir(csrc) if f.endswith(".cu"))
    for variant, extra in (("", list(extra_flags)), ("_prof", ["-DAA_PROF"] + list(extra_flags))):
        objs = []
        procs = []
        for cu in cus:
            o = os.path.join(EXP, f"{tag}{variant}_{cu}.o")
            procs.append(subprocess.Popen([nvcc] + flags + extra + ["-c", os.path.join(csrc, cu), "-o", o]))
            objs.append(o)
        for p in procs:
            assert p.wait() == 0
        subprocess.run([nvcc] + arch + ["-shared", "-o", os.path.join(EXP, f"lib{tag}{variant}.so")] + objs
                       + ["-lcuda"], check=True)
        for o in objs:
            os.unlink(o)


def main():
    rev = sys.argv[1] if len(sys.argv) > 1 else "HEAD"
    os.makedirs(EXP, exist_ok=True)
    wt = "/tmp/ab_worktree"
    if os.path.exists(wt):
        subprocess.run(["git", "-C", ROOT, "worktree", "remove", "--force", wt])
        shutil.rmtree(wt, ignore_errors=True)
    subprocess.run(["git", "-C", ROOT, "worktree", "add", "--detach", wt, rev], check=True,
                   stdout=subprocess.DEVNULL)
    try:
        build_tree(wt, "A")
    finally:
        subprocess.run(["git", "-C", ROOT, "worktree", "remove", "--force", wt])
    build_tree(ROOT, "B")
    # optional third variant: the working tree with extra nvcc flags (AB_C_FLAGS)
    cflags = os.environ.get("AB_C_FLAGS", "").split()
    if cflags:
        build_tree(ROOT, "C", cflags)
    print("built exp/libA.so exp/libB.so (+ _prof)" + (f", exp/libC.so ({' '.join(cflags)})" if cflags else ""))


if __name__ == "__main__":
    main()
