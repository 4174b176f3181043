#!/bin/bash
OUT=gpurun_out/r02split; mkdir -p $OUT
export PYTHONUNBUFFERED=1
MMAS_LIB=$PWD/tools/ab_split.so timeout 900 python -m pytest -x -q tests/test_parity_full_gpu.py tests/test_parity_gpu.py tests/test_fallback_compact_gpu.py -k "driver or c1 or small or compact or fused" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -2 $OUT/pytest.log
bash scripts/ab.sh r02split/c2 "--steps 20 --warmup 5" tools/ab_base.so tools/ab_split.so > /dev/null 2>&1
cat $OUT/c2/ab.txt
bash scripts/ab.sh r02split/c2s "--steps 300 --warmup 100" tools/ab_base.so tools/ab_split.so > /dev/null 2>&1
cat $OUT/c2s/ab.txt
