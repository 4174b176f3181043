mkdir -p gpurun_out/r02x
bash scripts/ab.sh r02x_c3 "--config C3 --steps 20 --warmup 5" abx/libmmas_c3v.so abx/libmmas_c3v.so@MMAS_FB_VARIANT=1 abx/libmmas_c3v.so@MMAS_FB_VARIANT=2
