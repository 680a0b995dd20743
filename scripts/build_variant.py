"""Build a library variant into variants/lib<name>.so: a copy of csrc/ with
files replaced (path=file pairs, e.g. normad_cl.cuh=/tmp/x.cuh or
normad_cl.cuh=git:HEAD) and extra nvcc flags -- for A/B on the GPU
(scripts/variants.sh)."""
import os, shutil, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_03637_b200 import build as b  # noqa: E402
name, rest = sys.argv[1], sys.argv[2:]
tmp = tempfile.mkdtemp()
src = os.path.join(tmp, "csrc")
shutil.copytree(os.path.join(ROOT, "paper_1711_03637_b200", "csrc"), src)
flags = []
for r in rest:
    if r.startswith("-"):
        flags.append(r)
        continue
    f, v = r.split("=", 1)
    dst = os.path.join(src, f)
    if v.startswith("git:"):
        txt = subprocess.run(["git", "-C", ROOT, "show", f"{v[4:]}:paper_1711_03637_b200/csrc/{f}"],
                             capture_output=True, text=True, check=True).stdout
        open(dst, "w").write(txt)
    else:
        shutil.copy(v, dst)
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
out = os.path.join(ROOT, "variants", f"lib{name}.so")
subprocess.run([b.nvcc(), *b.NVCC_FLAGS, *flags, "-I", os.path.join(ROOT, "include"), "-o", out,
                os.path.join(src, "snn_b200.cu")], check=True)
print(out)
