#!/bin/bash
# round-2 final evidence: the standard session (tests, smoke, every bench, ncu) + the
# bounds-checked parity suites
bash scripts/gpu_session.sh r02v6 facts tests smoke bench benchC1 benchC2x8 benchC3 benchC4 benchC4CT benchC5 benchC5L benchC65KL reference ncu ncuC4
timeout 1800 python tools/checked_runs.py -q > gpurun_out/r02v6/checked.log 2>&1; echo "checked rc=$?" >> gpurun_out/r02v6/checked.log
tail -2 gpurun_out/r02v6/checked.log
