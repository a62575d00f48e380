#!/bin/bash
# tops cap sweep (rows) on case9241: per-stage times
for T in 8 16 24 32; do echo "TOPS=$T $(RH_TOPS=$T timeout 300 python tools/diag.py case9241pegase 2>&1 | grep stages)"; done
