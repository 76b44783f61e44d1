"""Build librlx.so from the csrc/include of a git revision into a side file
(A/B kernel experiments on one box: tools/gpu_ab.sh).

    python tools/build_variant.py <rev> <out.so> [-DNAME=VALUE ...]
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rev, out = sys.argv[1], os.path.abspath(sys.argv[2])
defs = [a for a in sys.argv[3:] if a.startswith("-D")]
with tempfile.TemporaryDirectory() as tmp:
    for path in ("paper_2604_23838_b200/csrc", "paper_2604_23838_b200/build.py", "include"):
        arch = subprocess.run(["git", "-C", ROOT, "archive", rev, path], check=True, capture_output=True).stdout
        subprocess.run(["tar", "-x", "-C", tmp], input=arch, check=True)
    sys.path.insert(0, os.path.join(tmp, "paper_2604_23838_b200"))
    import build  # noqa: E402  (the revision's own build recipe)

    build.build(force=True, out=out, defines=tuple(d[2:] for d in defs))
print(out)
