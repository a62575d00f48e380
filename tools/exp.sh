for D in 0 1 3; do echo "RH_DEBUG=$D"; RH_DEBUG=$D timeout 300 python tools/diag.py case9241pegase 2>&1 | grep stages | sed 's/.*stages/stages/'; done
