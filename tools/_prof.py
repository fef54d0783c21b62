"""tools/: load the profiling build of the library (CGB_* environment knobs and the
CGB_DEBUG_SW stage switches are compiled only into libconvgemm_b200_prof.so).
Import this before paper_2005_06410_b200; builds the variant if it is missing."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
_PROF = os.path.join(ROOT, "paper_2005_06410_b200", "libconvgemm_b200_prof.so")
if not os.environ.get("CGB_LIB_OVERRIDE"):
    if not os.path.isdir("/root/reference") and not os.path.exists(_PROF):
        raise ImportError("libconvgemm_b200_prof.so missing: build it in the build container "
                          "(python paper_2005_06410_b200/build.py --profiling)")
    if os.path.isdir("/root/reference"):  # build container: (re)build when stale
        import importlib.util
        spec = importlib.util.spec_from_file_location("_cgb_build", os.path.join(ROOT, "paper_2005_06410_b200", "build.py"))
        b = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(b)
        b.build(profiling=True)
    os.environ["CGB_LIB_OVERRIDE"] = _PROF
