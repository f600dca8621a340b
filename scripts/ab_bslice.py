import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_12228_b200 import _build
LIBPATH = os.path.abspath(sys.argv[1])
_build.LIB = LIBPATH
_build.build = lambda *a, **k: LIBPATH
sys.argv = [sys.argv[0]] + sys.argv[2:]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_bslice.py")).read())
