mkdir -p gpurun_out/var4
export LMS_LAG=1
python tools/kk_variants.py variants/base.so variants/cfoside.so variants/base.so variants/cfoside.so > gpurun_out/var4/v.txt 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "chunking or randomised or c4 or large_history or realtime" > gpurun_out/var4/t.txt 2>&1
