"""(CPU or GPU box) Build a compile-time variant of liblce.so for A/B runs:

    python scripts/build_variant.py paper_2605_21442_b200/liblce_v1.so LCE_WAIT_HINT=1 [...]

then `LCE_LIB_PATH=<that .so> python bench.py ...` (scripts/ab_bench.sh)."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("lce_build", os.path.join(ROOT, "paper_2605_21442_b200", "build.py"))
mod = importlib.util.module_from_spec(spec)
spec.loader.exec_module(mod)
print(mod.build(force=True, dest=os.path.abspath(sys.argv[1]), defines=tuple(sys.argv[2:])))
