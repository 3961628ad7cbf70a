python - <<'PY'
import ctypes, os
from paper_2005_07132_b200 import fkk
PY
timeout 300 python tools/prof_transform.py 703026 3 2>&1 | grep -v Warn | tail -1 | grep -o "'gram': [0-9.]*"
FKK_GRAM_DBG=1 timeout 300 python tools/prof_transform.py 703026 1 2>&1 | grep "gram_pre2 dbg" | tail -1
timeout 900 python -m pytest tests -m gpu -q -x -k "cfg4 or gram" 2>&1 | tail -2
