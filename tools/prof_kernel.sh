#!/bin/bash
# Dev helper: ncu --set full of one launch of the kernel matching $2 in phase $3 of tools/time_phase.py -> gpurun_out/$1.ncu-rep
tag=$1; k=${2:-lz77}; ph=${3:-lz77}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 -o gpurun_out/$tag python tools/time_phase.py $ph > gpurun_out/$tag.log 2>&1; tail -2 gpurun_out/$tag.log
