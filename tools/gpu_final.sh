#!/bin/bash
# Round-end evidence pass: tests, bench lines for every config, ncu launch lists + full captures.
TAG=${1:-r01f}
bash tools/gpu_status.sh $TAG "c2 c1 c3 c4 c4v c5 c3r c3rs"
bash tools/gpu_profiles.sh r01 "c2 c1 c3 c4 c4v c5 c3r c3rs"
