timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k fused 2>&1 | tail -1
for cfg in "1 2 0" "1 3 0" "1 5 0" "2 8 0" "1 5 1" "1 5 7" "1 5 6" "1 4 7" "2 8 7" "3 11 7"; do set -- $cfg
DISPCORR_FUSED=1 DISPCORR_FUSED_LAG=$1 DISPCORR_FUSED_DEPTH=$2 DISPCORR_FUSED_HINTS=$3 timeout 120 python tools/debug/variant_bench.py 20 192 | python -c "import json,sys; d=json.load(sys.stdin); print('lag $1 depth $2 hints $3', round(d['GS/s'],1))"
done
