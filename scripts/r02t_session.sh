mkdir -p gpurun_out/r02t
timeout 900 python -m pytest tests/test_checkpoint_gpu.py tests/test_capi.py -m "gpu or not gpu" -q -x > gpurun_out/r02t/pytest.log 2>&1; echo rc=$? >> gpurun_out/r02t/pytest.log; tail -3 gpurun_out/r02t/pytest.log
for sc in weak strong; do
  MMAS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --scaling $sc --config C1 > gpurun_out/r02t/bench_n2_$sc.json 2> gpurun_out/r02t/bench_n2_$sc.err; echo "n2 $sc rc=$?"; head -c 400 gpurun_out/r02t/bench_n2_$sc.json; echo
done
MMAS_EXCHANGE=collective MMAS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 5 --warmup 3 --config C1 > gpurun_out/r02t/bench_n2_coll.json 2> gpurun_out/r02t/bench_n2_coll.err; echo "n2 collective rc=$?"; head -c 400 gpurun_out/r02t/bench_n2_coll.json; echo
