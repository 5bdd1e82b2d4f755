mkdir -p gpurun_out/var6
export LMS_LAG=1
python tools/kk_variants.py variants/cur.so variants/fused.so variants/cur.so variants/fused.so > gpurun_out/var6/v.txt 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c4 or c3 or chunking or randomised or sharded_kk or data_aided or wl or chain or large_history or c5" > gpurun_out/var6/t.txt 2>&1
