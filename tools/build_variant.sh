#!/bin/bash
# Build the engine with extra -D flags into tools/libvar_<name>.so (A/B experiments):
#   EXTRA="-DPP_NO_FLAT_ROWS" bash tools/build_variant.sh noflat
set -e
cd "$(dirname "$0")/.."
N=$1
mkdir -p build/var_$N
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden $EXTRA -Iinclude"
for f in pp_context pp_schedule pp_eval pp_eval_general pp_moves pp_npv pp_price pp_host pp_lns pp_vae pp_uncert; do
  nvcc $F -c paper_2511_18296_b200/csrc/$f.cu -o build/var_$N/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libvar_$N.so build/var_$N/*.o
