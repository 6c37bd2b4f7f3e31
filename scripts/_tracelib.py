"""Dev scripts that read the pipeline trace need a -DTAPER_TRACE=1 build of the library
(the product build compiles the probes out).  Importing this module builds that variant
into build/libtaper_trace.so once and points TAPER_LIB at it (unless TAPER_LIB is set)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
if "TAPER_LIB" not in os.environ:
    from paper_2605_06914_b200 import build as _b
    _out = os.path.join(ROOT, "build", "libtaper_trace.so")
    os.makedirs(os.path.dirname(_out), exist_ok=True)
    _b.build(force=True, defines=["TAPER_TRACE=1", *filter(None, os.environ.get("TAPER_EXTRA_DEFINES", "").split(","))],
             out=_out)
    os.environ["TAPER_LIB"] = _out
