# scratch GPU job: cull at 18M anchors (cold in L2) for ab/<variant> libraries
for V in "$@"; do
  echo "== $V"
  GSC_AB_LIB=$PWD/ab/$V/libgscache.so PYTHONPATH=. timeout 900 python -c "
import os, sys
from paper_2502_14938_b200 import _abi
_abi.SO_PATH = os.environ['GSC_AB_LIB']
sys.argv = ['cull_scale.py', '18000000', '40']
import runpy; runpy.run_path('tools/cull_scale.py', run_name='__main__')"
done
