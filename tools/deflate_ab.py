"""A/B of library variants on tools/deflate_probe.py's workload.
    python tools/deflate_ab.py <workload> variants/a.so ..."""
import runpy
import sys

sys.path.insert(0, ".")
from paper_1703_02438_b200 import _native as N  # noqa: E402

wl = sys.argv[1]
for path in [None] + sys.argv[2:]:
    N._lib = N.load(path) if path else N.load()
    print("==", path or "in-tree", flush=True)
    sys.argv = ["tools/deflate_probe.py", wl]
    runpy.run_path("tools/deflate_probe.py", run_name="__main__")
