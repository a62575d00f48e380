#!/bin/bash
CASE=${1:-case9241pegase}
for CPL in 1 2; do for R in 128 256 512; do
  echo "CPL=$CPL RMAX=$R $(RH_CPL=$CPL RH_RMAX=$R timeout 300 python tools/diag.py $CASE 2>&1 | grep stages | sed 's/grad.*full H/full H/')"
done; done
