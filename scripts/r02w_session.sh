mkdir -p gpurun_out/r02w
bash scripts/ab.sh r02w_c2 "--steps 20 --warmup 5" abx/libmmas_pf2.so abx/libmmas_l1pf.so abx/libmmas_l1pf.so@MMAS_FB_L1PF=0
bash scripts/ab.sh r02w_c1 "--config C1 --steps 50 --warmup 5" abx/libmmas_pf2.so abx/libmmas_l1pf.so
