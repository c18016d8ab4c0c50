"""A/B of library variants on tools/inflate_probe.py's workload.
    python tools/inflate_ab.py variants/a.so ..."""
import runpy
import sys

sys.path.insert(0, ".")
from paper_1703_02438_b200 import _native as N  # noqa: E402

for path in [None] + sys.argv[1:]:
    N._lib = N.load(path) if path else N.load()
    print("==", path or "in-tree", flush=True)
    runpy.run_path("tools/inflate_probe.py", run_name="__main__")
