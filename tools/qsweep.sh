# bulk-quantize variants (compile defines) timed by tools/qbench.py:
#   bash tools/qsweep.sh "" "NQKV_Q_CTAS_PER_SM=4" ...
for spec in "$@"; do
  python - "$spec" <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2505_16210_b200 import build as bld
spec = sys.argv[1]
defs = dict(kv.split("=") for kv in spec.split(",")) if spec else {}
bld.build_variant("/tmp/libnqkv_q.so", defs)
PY
  echo "== $spec"; NQKV_LIB=/tmp/libnqkv_q.so python tools/qbench.py
done
