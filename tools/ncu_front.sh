#!/bin/bash
# ncu capture of the fused router front at c2 (tools/front_time.py drives it)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:route_front -c 1 -o gpurun_out/front_${1:-v} -f \
    python tools/front_time.py > gpurun_out/ncu_front.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:route_front -c 3 python tools/front_time.py \
    >> gpurun_out/ncu_front.log 2>&1
