#!/bin/bash
# One GPU session: parity tests, bench, launch list, full ncu capture of the
# dominant kernel.  Outputs land in gpurun_out/ (scratch); summaries are copied
# into profiles/ by hand.
set -u
mkdir -p gpurun_out
TAG=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
if [ "${SKIP_TESTS:-0}" = "0" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -3 gpurun_out/${TAG}_pytest.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
if [ "${SKIP_NCU:-0}" = "0" ]; then
  timeout 300 python tools/quick_time.py c4_tau > gpurun_out/${TAG}_qt.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:kin_jit_stoch|stochastic_kernel" -s 1 -c 1 \
      -o gpurun_out/${TAG}_tau python tools/quick_time.py c4_tau > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
