mkdir -p gpurun_out/r02u
bash scripts/ab.sh r02u_c2 "--steps 20 --warmup 5" abx/libmmas_noinl.so abx/libmmas_fbv.so abx/libmmas_fbv.so@MMAS_FB_VARIANT=1 abx/libmmas_fbv.so@MMAS_FB_VARIANT=2
bash scripts/ab.sh r02u_c1 "--config C1 --steps 50 --warmup 5" abx/libmmas_noinl.so abx/libmmas_fbv.so@MMAS_FB_VARIANT=1 abx/libmmas_fbv.so@MMAS_FB_VARIANT=2
