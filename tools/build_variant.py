"""Build libcoop.so with one csrc file swapped for a variant (kernel A/B experiments).

usage: python tools/build_variant.py <variant file> <name> [csrc file it replaces, default
       coop_search.cu]   ->  variants/<name>.so
Run the bench against it with COOP_LIB_OVERRIDE=variants/<name>.so.
"""
import glob, os, shutil, subprocess, sys, tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2311_00591_b200"))
import _build  # noqa: E402

src, name = sys.argv[1], sys.argv[2]
target = sys.argv[3] if len(sys.argv) > 3 else "coop_search.cu"
tmp = tempfile.mkdtemp()
for f in glob.glob(os.path.join(ROOT, "paper_2311_00591_b200", "csrc", "*")):
    shutil.copy(f, tmp)
shutil.copy(src, os.path.join(tmp, target))
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
out = os.path.join(ROOT, "variants", name + ".so")
subprocess.run([_build.NVCC, *_build.NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", tmp,
                "-o", out, *sorted(glob.glob(os.path.join(tmp, "*.cu")))], check=True)
print(out)
