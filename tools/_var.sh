mkdir -p gpurun_out/var3
export LMS_LAG=1
python tools/kk_variants.py variants/base.so variants/magic.so variants/cfo3r104.so variants/magic_cfo.so > gpurun_out/var3/v.txt 2>&1
