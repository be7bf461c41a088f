"""tools/time_graph_gaps.py with the library given as argv[1] (experiment variants)."""
import sys
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib
_lib.load(sys.argv[1])
import runpy
runpy.run_path('tools/time_graph_gaps.py', run_name='__main__')
