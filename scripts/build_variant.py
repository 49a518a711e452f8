"""Build a profiling variant of libnent_b200.so into scripts/_bin/ with extra
nvcc defines, e.g. `python scripts/build_variant.py timers -DNENT_TC05_TIMERS`.
`--only a,b` recompiles just csrc/a.cu and csrc/b.cu with the defines and links
the release objects (paper_1509_03838_b200/_obj) for everything else."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _build as B  # noqa: E402

args = sys.argv[1:]
only = None
if "--only" in args:
    i = args.index("--only")
    only = set(args[i + 1].split(","))
    del args[i:i + 2]
name, defs = args[0], args[1:]
out = Path(__file__).resolve().parent / "_bin"
out.mkdir(exist_ok=True)
obj = Path("/tmp") / f"nent_variant_obj_{name}"  # objects stay out of the gpurun snapshot
obj.mkdir(parents=True, exist_ok=True)
nvcc = B._nvcc()
if only is not None:
    B.build()  # release objects up to date


def one(src):
    if only is not None and src.stem not in only:
        return B.OBJ / (src.stem + ".o")
    o = obj / (src.stem + ".o")
    subprocess.run([nvcc, *B.NVCC_FLAGS, *defs, "-c", str(src), "-o", str(o)], check=True)
    return o


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, sorted(B.CSRC.glob("*.cu"))))
subprocess.run([nvcc, *B.ARCH, "-shared", "-cudart", "static", "-o", str(out / f"libnent_b200_{name}.so"),
                *map(str, objs), "-lrt", "-ldl", "-lpthread"], check=True)
print(out / f"libnent_b200_{name}.so")
