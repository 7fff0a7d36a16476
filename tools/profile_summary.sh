#!/bin/bash
# Summarise one gpu_round.sh capture (gpurun_out/<TAG>_*) into profiles/<TAG>_*.
set -eu
TAG=$1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > profiles/${TAG}_launches_summary.txt
ncu -i gpurun_out/${TAG}_tau.ncu-rep --page raw --csv 2>/dev/null > /tmp/${TAG}_raw.csv
python tools/ncu_raw_summary.py /tmp/${TAG}_raw.csv > profiles/${TAG}_tau_ncu_raw.txt
ncu -i gpurun_out/${TAG}_tau.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/${TAG}_sass.csv
python tools/ncu_sass_summary.py /tmp/${TAG}_sass.csv > profiles/${TAG}_tau_sass_summary.txt
cp gpurun_out/${TAG}_bench.json profiles/${TAG}_bench.json
