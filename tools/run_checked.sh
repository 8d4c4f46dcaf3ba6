#!/bin/bash
# Memory-safety run of the GPU suite against the checked library (the compute-sanitizer stand-in:
# guard zones around every device buffer, 0xFF-filled fresh payloads, device-side PP_DCHECK traps).
# Build here first: python -c 'import __graft_entry__ as g; g.build_checked()'
cd "$(dirname "$0")/.."
export PP_LIB="$PWD/paper_2511_18296_b200/libpitplan_b200_checked.so"
test -f "$PP_LIB" || { echo "missing $PP_LIB"; exit 2; }
python -m pytest tests -q -m gpu -p no:cacheprovider "$@"
