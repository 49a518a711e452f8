"""Build libnent_b200_<name>.so in scripts/_bin/ with ONE translation unit taken from another
commit (its .cu and every csrc header as of that commit), the rest from the release objects:
`python scripts/build_at_commit.py NAME COMMIT conv_tc05_m3 [nvcc defines...]` -- for same-box A/B."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _build as B  # noqa: E402

name, commit, stem, defs = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:]
root = Path(__file__).resolve().parents[1]
src = Path("/tmp") / f"nent_src_{name}" / "a" / "b"  # (the sources include ../../include/nent_b200.h)
src.mkdir(parents=True, exist_ok=True)
inc = src.parents[1] / "include"
inc.mkdir(exist_ok=True)
(inc / "nent_b200.h").write_bytes((root / "include" / "nent_b200.h").read_bytes())
rel = B.CSRC.relative_to(root)
files = subprocess.run(["git", "ls-tree", "--name-only", commit, str(rel) + "/"], cwd=root, check=True,
                       capture_output=True, text=True).stdout.split()
for f in files:
    (src / Path(f).name).write_bytes(subprocess.run(["git", "show", f"{commit}:{f}"], cwd=root, check=True,
                                                    capture_output=True).stdout)
B.build()
obj = src / (stem + ".o")
subprocess.run([B._nvcc(), *B.NVCC_FLAGS, *defs, "-c", str(src / (stem + ".cu")), "-o", str(obj)], check=True)
objs = [obj if o.stem == stem else o for o in sorted(B.OBJ.glob("*.o"))]
out = root / "scripts" / "_bin" / f"libnent_b200_{name}.so"
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-cudart", "static", "-o", str(out), *map(str, objs), "-lrt", "-ldl", "-lpthread"],
               check=True)
print(out)
