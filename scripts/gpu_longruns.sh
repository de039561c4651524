#!/bin/bash
# Validation runs: the plunging foil's full plunge cycles on the production
# mesh M1 and the cylinder at 32 cells per diameter.  Usage (under gpurun):
#   bash scripts/gpu_longruns.sh foil [cycles] [max-minutes]   |   bash scripts/gpu_longruns.sh cylinder
mkdir -p gpurun_out
case "${1:-foil}" in
  foil) python scripts/production_cycles.py --cycles ${2:-3} --max-minutes ${3:-150} --out-prefix gpurun_out/f1_M1 \
          > gpurun_out/f1_M1.log 2>&1; tail -c 3000 gpurun_out/f1_M1.log ;;
  cylinder) timeout 1500 python scripts/validate_cylinder.py --nx 1024 --ny 768 --dt 0.01 --steps 8000 --omega-p 1.98 \
          --maxit-p 30000 --out gpurun_out/cylinder_1024x768 > gpurun_out/cyl1024.log 2>&1; tail -c 1500 gpurun_out/cyl1024.log ;;
esac
