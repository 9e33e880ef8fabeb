"""python tools/exp/run_lib.py LIB SCRIPT ARGS...: run SCRIPT with libsdcsw replaced by LIB."""
import runpy
import sys
sys.path.insert(0, '/root/repo')
from paper_2403_20135_b200 import _native
_native.LIB_PATH = sys.argv[1]
_native.load(_native.LIB_PATH)
script = sys.argv[2]
sys.argv = [script] + sys.argv[3:]
runpy.run_path(script, run_name='__main__')
