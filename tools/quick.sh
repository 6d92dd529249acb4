#!/bin/bash
# Quick GPU check: parity tests + bench (no cpu baseline) + launch list.
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest.txt
tail -15 $OUT/pytest.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; tail -3 $OUT/bench.err
python -c "import json; d=json.load(open('$OUT/bench.json')); print(d['ms_per_step'], d['phases_us'], d['value'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py $OUT/launches.csv | head -25
python tools/host_overhead.py
MK_HOST_TIMING=1 python tools/host_overhead.py 2>&1 | grep "mk host" | tail -6
