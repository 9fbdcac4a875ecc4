# A/B of bench.py ms_per_step between the in-tree library and a compile-define
# variant (interleaved):  bash tools/ab_variant.sh "NQKV_X=1,NQKV_Y=2"
python - "$1" <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2505_16210_b200 import build as bld
defs = dict(kv.split("=") for kv in sys.argv[1].split(","))
bld.build_variant("/tmp/libnqkv_ab.so", defs)
PY
for i in 1 2; do for lib in "" /tmp/libnqkv_ab.so; do
  r=$(NQKV_LIB=$lib python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['mean_launch_us'])")
  echo "lib=${lib:-in-tree} $r"
done; done
