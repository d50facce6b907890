timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "largest_pulses" > gpurun_out/s2_test21.log 2>&1
for pipe in 0 1; do for mb in 16 32 48 64 128 512; do
 echo "pipe $pipe mb $mb $(DISPCORR_PIPE=$pipe DISPCORR_CHUNK_MB=$mb timeout 120 python tools/debug/variant_bench.py 20 256 2>&1 | tail -1)"
done; done > gpurun_out/s2_sweep.log 2>&1
