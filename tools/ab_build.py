"""Build the library from the sources of a git revision (or the working tree,
REV = "wt") into paper_2006_13188_b200/lib/ab/NAME.so, for A/B kernel timing
with XCB_LIB_OVERRIDE (tools/ab_kernels.py).

  AB_DEFS="-DNAME=VALUE ..." python tools/ab_build.py REV NAME
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_13188_b200 import build as B  # noqa: E402

rev, name = sys.argv[1], sys.argv[2]
tree = f"/tmp/ab_{name}"
shutil.rmtree(tree, ignore_errors=True)
os.makedirs(tree)
if rev == "wt":
    shutil.copytree(os.path.join(ROOT, "paper_2006_13188_b200", "csrc"),
                    os.path.join(tree, "paper_2006_13188_b200", "csrc"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tree, "include"))
else:
    arc = subprocess.run(["git", "-C", ROOT, "archive", rev, "paper_2006_13188_b200/csrc",
                          "include"], capture_output=True, check=True).stdout
    subprocess.run(["tar", "-x", "-C", tree], input=arc, check=True)
csrc = os.path.join(tree, "paper_2006_13188_b200", "csrc")
flags = [f if f != os.path.join(ROOT, "include") else os.path.join(tree, "include")
         for f in B.FLAGS] + os.environ.get("AB_DEFS", "").split()  # e.g. -DXCB_PLAN_1152=...
srcs = [s for s in os.listdir(csrc) if s.endswith((".cu", ".cpp"))]


def comp(s):
    obj = os.path.join(tree, s + ".o")
    subprocess.run([B._nvcc(), *flags, "-c", os.path.join(csrc, s), "-o", obj], check=True)
    return obj


with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
    objs = list(ex.map(comp, srcs))
out = os.path.join(ROOT, "paper_2006_13188_b200", "lib", "ab", name + ".so")
os.makedirs(os.path.dirname(out), exist_ok=True)
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", out, *objs], check=True)
print(out)
