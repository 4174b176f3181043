#!/bin/bash
# One GPU session: device facts, parity tests, smoke, benches, ncu launch list + full captures.
# Usage (from the repo root, under gpurun): bash scripts/gpu_session.sh [tag] [what...]
TAG=${1:-r01}
shift || true
WHAT=${@:-"facts tests smoke bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONUNBUFFERED=1
has() { [[ " $WHAT " == *" $1 "* ]]; }
if has facts; then
  nvidia-smi > $OUT/nvidia-smi.txt 2>&1
  nvidia-smi -q -d CLOCK >> $OUT/nvidia-smi.txt 2>&1
  nproc > $OUT/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $OUT/nproc.txt
  python -c "import torch; p=torch.cuda.get_device_properties(0); print(p); print('sms',p.multi_processor_count,'l2',p.L2_cache_size)" > $OUT/device.txt 2>&1
fi
if has tests; then
  timeout 1500 python -m pytest tests -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
if has smoke; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
  tail -2 $OUT/smoke.log
fi
if has bench; then
  # the driver's command (iterations 5-24) and the default (steady state, 1000 steps)
  timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_driver.json 2> $OUT/bench_driver.err; echo "bench rc=$?" >> $OUT/bench_driver.err
  head -c 400 $OUT/bench_driver.json; echo
  MMAS_CREATE_PROFILE=1 timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
  head -c 400 $OUT/bench.json; echo
fi
for cfg in C1 C3 C4 C4CT C5 C5L C65KL C2x8 C2RWM C4RWM C4RWMCT; do
  if has bench$cfg; then
    steps=50; [[ $cfg == C4* ]] && steps=20; [[ $cfg == C5* ]] && steps=6; [ $cfg == C65KL ] && steps=3
    [ $cfg == C2RWM ] && steps=200; [ $cfg == C2x8 ] && steps=20
    timeout 1200 python bench.py --config $cfg --steps $steps --warmup 5 --no-cpu-baseline > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err
    head -c 300 $OUT/bench_$cfg.json; echo
  fi
done
if has reference; then
  timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
  cat $OUT/bench_reference.json
fi
# summarise a capture on the box (text summary + per-launch json); keep the report only if
# KEEP_REPS=1 (gpurun copies back at most 64 MiB)
digest() {  # digest CONFIG KERNEL REPORT_BASENAME
  if [ -f $OUT/$3.ncu-rep ]; then
    python scripts/ncu_summary.py $OUT/$3.ncu-rep 40 > $OUT/$3.txt 2>&1
    python scripts/ncu_json.py --out $OUT/ncu_traffic.json $1:$2:$OUT/$3.ncu-rep > /dev/null 2>&1
    [ "${KEEP_REPS:-0}" == 1 ] || rm -f $OUT/$3.ncu-rep
  fi
}
L2M="lts__t_bytes.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum"
if has ncu; then
  # the driver's bench command (iterations 5-24 timed)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
     python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/ncu_launches_bench.log 2>&1
  # construction in the driver's window (iteration 10) and at steady state (iteration 400)
  timeout 900 ncu --set full --metrics $L2M --clock-control none --import-source on -k regex:construct -s 10 -c 1 \
     -o $OUT/prof_construct_C2_it10 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/ncu_full_construct10.log 2>&1
  digest C2@10 construct_cl_kernel prof_construct_C2_it10
  timeout 900 ncu --set full --metrics $L2M --clock-control none --import-source on -k regex:construct -s 400 -c 1 \
     -o $OUT/prof_construct_C2_it400 python bench.py --steps 420 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_construct.log 2>&1
  digest C2@400 construct_cl_kernel prof_construct_C2_it400
  # C2 fuses the update into the construction launch; the stand-alone update kernel is
  # captured from the A/B path (--separate-update)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pheromone_update -s 400 -c 1 -o $OUT/prof_update_C2 \
     python bench.py --steps 420 --warmup 3 --no-cpu-baseline --separate-update > $OUT/ncu_full_update.log 2>&1
  digest C2 pheromone_update_kernel prof_update_C2
  ls -la $OUT
fi
for cfg in C1 C3 C4 C4CT C2RWM C4RWM C4RWMCT C5 C5L C2x8; do
  if has ncu$cfg; then
    timeout 900 ncu --set full --metrics $L2M --clock-control none --import-source on -k regex:construct -s 5 -c 1 -o $OUT/prof_construct_$cfg \
       python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_construct_$cfg.log 2>&1
    kern=construct_cl_kernel
    case $cfg in C4) kern=construct_full_kernel;; C4CT) kern=construct_ct_kernel;; *RWM*) kern=construct_rwm_kernel;; esac
    digest $cfg@5 $kern prof_construct_$cfg
  fi
done
if has ncuC5; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:two_opt -s 2 -c 1 -o $OUT/prof_two_opt_C5 \
     python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_two_opt.log 2>&1
  digest C5 two_opt_coop_kernel prof_two_opt_C5
fi
