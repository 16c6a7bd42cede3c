#!/bin/bash
# The GPU suite on the bounds-checked library (build.py --checked: SGL_DCHECK on
# every grid / TMA / output index of the window kernels) -- the stand-in for
# compute-sanitizer memcheck, which is closed on this GPU pool.
out=${1:-gpurun_out}
python -m paper_1809_10786_b200.build --checked > /dev/null
SGL_LIBRARY=$PWD/paper_1809_10786_b200/_lib/libsgl_b200_checked.so \
  python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > $out/checked_suite.log
SGL_LIBRARY=$PWD/paper_1809_10786_b200/_lib/libsgl_b200_checked.so python -c "
import ctypes, os
from paper_1809_10786_b200 import _native
print('loaded', _native.LIB_PATH)
" >> $out/checked_suite.log 2>&1
grep -c SGL_CHECKED $out/checked_suite.log
tail -3 $out/checked_suite.log
