"""Build a variant of libmoirai_b200.so with extra nvcc defines for an A/B on the GPU box:
    python scripts/build_variant.py NAME -DMP_FOO=1 ...  ->  build/variants/NAME/libmoirai_b200.so
(mp_eval.cu recompiled with the defines, the other objects reused from the in-tree build;
select it with MOIRAI_B200_LIB=build/variants/NAME/libmoirai_b200.so, see scripts/abv.sh)."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2312_04025_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
B.build()
out = B.ROOT / "build" / "variants" / name
out.mkdir(parents=True, exist_ok=True)
obj = out / "mp_eval.o"
subprocess.run([B.nvcc(), *B.ARCH, *B.NVFLAGS, *defs, "-c", str(B.CSRC / "mp_eval.cu"), "-o", str(obj)], check=True)
objs = [obj] + [B.OBJ / (Path(s).stem + ".o") for s in B.SOURCES if s != "mp_eval.cu"]
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(out / "libmoirai_b200.so"), *map(str, objs),
                "-lcudart_static", "-lrt", "-lpthread", "-ldl"], check=True)
(out / "defines.txt").write_text(" ".join(defs) + "\n")
print(out / "libmoirai_b200.so")
