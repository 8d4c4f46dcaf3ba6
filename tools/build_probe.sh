#!/bin/bash
# Build the engine with globaltimer stage probes (tools/libprobe.so) for tools/step_timeline.py.
set -e
cd "$(dirname "$0")/.."
mkdir -p build/probe
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -DPP_EVAL_PROBE $EXTRA -Iinclude"
for f in pp_context pp_schedule pp_eval pp_eval_general pp_moves pp_npv pp_price pp_host pp_lns pp_vae pp_uncert; do
  nvcc $F -c paper_2511_18296_b200/csrc/$f.cu -o build/probe/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libprobe${SUFFIX}.so build/probe/*.o
