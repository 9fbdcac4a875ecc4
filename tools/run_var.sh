for cfg in "1 148 64 16384" "1 148 128 8192"; do
for d in "" "NQKV_PF=1" "NQKV_PF=2" "NQKV_PF=4"; do
echo "== $cfg DEFS=$d"
DEFS=$d python tools/trace_decode.py $cfg 2>&1 | grep -E "consumer +(full0|loop end)"
done; done
