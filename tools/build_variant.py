"""Build an A/B copy of the CUDA library with extra nvcc defines (timing experiments only).

  python tools/build_variant.py TAG -DNAME=VALUE ...

Writes paper_1905_04975_b200/libsn_b200_TAG.so (git-ignored; it travels to the GPU box); load it
with SN_LIB_PATH=<that path> (the binding then never rebuilds)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_04975_b200 as sn  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "paper_1905_04975_b200", "libsn_b200_%s.so" % tag)
cmd = ["nvcc", *sn.NVCC_FLAGS, *defs, "-shared", "-I", os.path.join(ROOT, "include"), "-o", out, *sn.sources()]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-4000:])
for line in r.stderr.splitlines():
    if "window_kernel" in line:
        i = r.stderr.splitlines().index(line)
        print("\n".join(r.stderr.splitlines()[i:i + 3]))
        break
print(out)
