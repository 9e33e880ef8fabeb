import sys
sys.path.insert(0, '/root/repo')
from paper_2403_20135_b200 import _native
_native.LIB_PATH = sys.argv[1]
_native.load(_native.LIB_PATH)
sys.argv = [sys.argv[0]] + sys.argv[2:]
import runpy
runpy.run_path('/root/repo/tools/stage_bench.py', run_name='__main__')
