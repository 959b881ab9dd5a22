#!/bin/bash
# K1 diagnostics: per-phase clock stamps (diagnostics build) and one ncu --set full capture of the
# projection kernel on the C5 element type. usage: bash tools/gpu_k1diag.sh TAG
TAG=${1:-k1d}
bash tools/phase_run.sh $TAG
bash tools/gpu_ncu.sh $TAG project_kernel
