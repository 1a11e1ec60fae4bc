"""Build a variant of libsem_b200.so with extra nvcc flags into
_exp/<name>/ (a copy of the package, include/ and semgen/), for A/B timing:
`PYTHONPATH=_exp/<name> python tools/ab_ops.py`.  Developer tool.
usage: python tools/ab_build.py NAME "-DFLAG=1 ..." """
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name, flags = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
dst = os.path.join(ROOT, "_exp", name)
if os.path.exists(dst):
    shutil.rmtree(dst)
os.makedirs(dst)
for d in ("paper_2405_05640_b200", "include", "semgen"):
    shutil.copytree(os.path.join(ROOT, d), os.path.join(dst, d),
                    ignore=shutil.ignore_patterns("build_obj", "*.so", "__pycache__"))
env = dict(os.environ, SEM_NVCC_EXTRA=flags)
subprocess.run([sys.executable, "-c", "from paper_2405_05640_b200 import build; build.build(force=True)"],
               cwd=dst, env=env, check=True)
print("built", dst)
