mkdir -p gpurun_out/r02y
bash scripts/ab.sh r02y_c5 "--config C5 --steps 3 --warmup 3" abx/libmmas_lspf.so abx/libmmas_lspf.so@MMAS_LS_PF=1
