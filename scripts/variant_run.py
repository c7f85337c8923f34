"""Run a repo script against a library variant built by scripts/variant.sh:
  python scripts/variant_run.py <variant> <script.py> [args...]
The variant's package directory goes first on sys.path, so `import
paper_2111_05894_b200` (and its libtiergraph_b200.so) resolves to the variant."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
var, script = sys.argv[1], sys.argv[2]
sys.argv = [script] + sys.argv[3:]
src = open(os.path.join(ROOT, script)).read()
sys.path.insert(0, ROOT)  # bench.py, oracle
sys.path.insert(0, os.path.join(ROOT, "variants", var))
import paper_2111_05894_b200 as P  # noqa: E402
print("package from", os.path.dirname(P.__file__), flush=True)
exec(compile(src, script, "exec"), {"__name__": "__main__", "__file__": os.path.join(ROOT, script)})
