#!/bin/bash
for R in 512 256; do echo "RMAX=$R"; RH_RMAX=$R timeout 300 python tools/diag.py case2869pegase case9241pegase 2>&1 | grep -v "^case" ; done
