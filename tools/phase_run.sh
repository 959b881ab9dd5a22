#!/bin/bash
# Phase breakdown of the flux kernel (clock64 stamps, ES_PHASE_TIMING) on the C5 element type.
mkdir -p gpurun_out
# the stamps are compiled in only with ES_STAMPS=1: rebuild a diagnostics library in a copy
cp paper_2312_07874_b200/libes_b200.so /tmp/libes_b200.so.prod
ES_STAMPS=1 python tools/build.py --force > gpurun_out/${1:-ph}_build.log 2>&1
ES_PHASE_TIMING=1 timeout 300 python tools/profile_run.py 3 12 8 3 > gpurun_out/${1:-ph}_phase.log 2>&1
cat gpurun_out/${1:-ph}_phase.log | tail -4
cp /tmp/libes_b200.so.prod paper_2312_07874_b200/libes_b200.so
