for mb in 2048 4096 8192; do
 echo "mb $mb $(DISPCORR_CHUNK_MB=$mb timeout 120 python tools/debug/variant_bench.py 20 1024 2>&1 | tail -1)"
done > gpurun_out/s52.log 2>&1
