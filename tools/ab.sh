#!/bin/bash
# A/B of libcf_base.so (previous build) vs libcf.so (current) on the same box, interleaved;
# extra args: flag lists for the current build (default 0,1)
FL=${1:-0,1}
for i in 1 2; do
  echo -n "base: "; CF_LIB=libcf_base.so python tools/driver_cost.py cfg3 0,1 2>&1 | grep flags | tr '\n' ' '; echo
  echo -n "new:  "; python tools/driver_cost.py cfg3 $FL 2>&1 | grep flags | tr '\n' ' '; echo
done
