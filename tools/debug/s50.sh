for mb in 256 512 1024 2048; do
 echo "mb $mb $(DISPCORR_CHUNK_MB=$mb timeout 120 python tools/debug/variant_bench.py 20 512 2>&1 | tail -1)"
done > gpurun_out/s50.log 2>&1
