# graph-chain per-layer time (tools/trace_chain.py NOTRACE=1 GRAPH=1) for the
# in-tree build and variant libraries, interleaved:  bash tools/ab_chain.sh lib.so ...
CFG=${CFG:-"8 32 64 2048 24"}
for i in 1 2; do for lib in "" "$@"; do
  r=$(NQKV_LIB=$lib NOTRACE=1 GRAPH=1 EARLY=${EARLY:-1} python tools/trace_chain.py $CFG 2>&1 | grep "graph chain")
  echo "${lib:-in-tree} $r"
done; done
if [ -d _ab/head ]; then for i in 1 2; do
  r=$(cd _ab/head && NOTRACE=1 GRAPH=1 python tools/trace_chain.py $CFG 2>&1 | grep "graph chain"); echo "head $r"; done; fi
