#!/bin/bash
# Phase breakdown of the flux kernel (clock64 stamps, ES_PHASE_TIMING) on the C5 element type.
mkdir -p gpurun_out
ES_PHASE_TIMING=1 timeout 300 python tools/profile_run.py 3 12 8 3 > gpurun_out/${1:-ph}_phase.log 2>&1
cat gpurun_out/${1:-ph}_phase.log | tail -4
