"""Build an A/B variant of libsdv2.so from a patched copy of csrc/ (measurement only; the
in-tree sources are untouched).  Usage:
  python tools/build_variant.py NAME [-DMACRO=VAL ...] [--sub 'file::old::new' ...]
writes paper_2511_07399_b200/variants/libsdv2_NAME.so (bench.py --lib / tools/ab.sh)."""
import os, shutil, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2511_07399_b200")
name, args = sys.argv[1], sys.argv[2:]
defs = [a for a in args if a.startswith("-D")]
subs = [args[i + 1] for i, a in enumerate(args) if a == "--sub"]
tmp = tempfile.mkdtemp()
shutil.copytree(os.path.join(PKG, "csrc"), os.path.join(tmp, "pkg", "csrc"))
shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
for s in subs:
    f, old, new = s.split("::")
    p = os.path.join(tmp, "pkg", "csrc", f)
    src = open(p).read()
    assert old in src, (f, old)
    open(p, "w").write(src.replace(old, new))
c = os.path.join(tmp, "pkg", "csrc")
out = os.path.join(PKG, "variants", f"libsdv2_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3", "-lineinfo",
       "-shared", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", *defs, "-o", out, os.path.join(c, "sdv2.cu"),
       os.path.join(c, "ctl.cpp"), os.path.join(c, "ctl_abi.cpp"), os.path.join(c, "slo.cpp"), os.path.join(c, "balance.cpp")]
subprocess.check_call(cmd)
print(out)
