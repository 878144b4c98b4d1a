#!/bin/bash
TAG=${1:-q}
bash tools/gpu_quick.sh $TAG
bash tools/gpu_ncu.sh $TAG k_rows_full C2
