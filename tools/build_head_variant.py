"""Build the library from a committed revision's kernel sources (default
git HEAD) as an A/B variant, build/variants/<name>/libgmi_b200.so, for
tools/ab_variants.sh.
    python tools/build_head_variant.py [name] [rev]"""
import os
import subprocess
import sys
import tempfile

sys.path.insert(0, os.getcwd())
import paper_2012_13257_b200._build as b  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "head"
rev = sys.argv[2] if len(sys.argv) > 2 else "HEAD"
with tempfile.TemporaryDirectory() as tmp:
    files = subprocess.run(["git", "ls-files", "paper_2012_13257_b200/csrc"], capture_output=True,
                           text=True, check=True).stdout.split()
    for f in files:
        os.makedirs(os.path.join(tmp, os.path.dirname(f)), exist_ok=True)
        with open(os.path.join(tmp, f), "w") as fh:
            fh.write(subprocess.run(["git", "show", f"{rev}:{f}"], capture_output=True, text=True,
                                    check=True).stdout)
    src = os.path.join(tmp, "paper_2012_13257_b200", "csrc")
    out = os.path.join(b.ROOT, "build", "variants", name)
    os.makedirs(out, exist_ok=True)
    subprocess.run(["nvcc", *b.NVCC_FLAGS, *b.ARCH, "-shared", f"-I{b.INCLUDE}", f"-I{src}",
                    *[os.path.join(src, s) for s in b.CU_SOURCES], "-o",
                    os.path.join(out, "libgmi_b200.so")], check=True)
print("built", name, "from", rev)
