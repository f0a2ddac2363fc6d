#!/bin/bash
# One measurement set on the GPU box: GPU tests, bench lines, the ncu launch list of the bench
# command, and one ncu --set full capture of an eager c2 step (per-kernel DRAM traffic).
# Large reports stay in /tmp; gpurun_out/ only gets summaries (its merge-back limit is 64 MiB).
#   tools/round_profile.sh TAG [skip-tests]
tag=${1:-v}
mkdir -p gpurun_out
if [ -z "$2" ]; then
  timeout 1200 python -m pytest tests -m gpu -q 2>&1 | grep -E "FAILED|ERROR|passed|failed|Error" | head -40 \
      > gpurun_out/gputest_$tag.log
  timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1
fi
timeout 600 python bench.py > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1_$tag.json 2> gpurun_out/bench_c1_$tag.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
n=$(python tools/profile_step.py 1 | sed -n 's/.*launches\/step \([0-9]*\).*/\1/p')
timeout 900 ncu --set full --import-source on --clock-control none --launch-skip $n -o /tmp/step_$tag -f \
    python tools/profile_step.py 2 > gpurun_out/profile_step_$tag.log 2>&1
python tools/ncu_traffic.py /tmp/step_$tag.ncu-rep gpurun_out/step_tags.json gpurun_out/ncu_traffic_$tag.json \
    >> gpurun_out/profile_step_$tag.log 2>&1
ncu -i /tmp/step_$tag.ncu-rep --page raw --csv > gpurun_out/step_raw_$tag.csv 2>/dev/null
sz=$(stat -c %s /tmp/step_$tag.ncu-rep 2>/dev/null || echo 0)
[ "$sz" -lt 40000000 ] && cp /tmp/step_$tag.ncu-rep gpurun_out/
tail -3 gpurun_out/gputest_$tag.log 2>/dev/null; tail -1 gpurun_out/smoke_$tag.log 2>/dev/null
