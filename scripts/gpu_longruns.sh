#!/bin/bash
# Validation runs: the plunging foil's full plunge cycles on the production
# mesh M1 and the cylinder at 32 cells per diameter.  A gpurun call is capped at 60 minutes, so the
# foil run goes in segments: each resumes from ckpt/f1_M1.npz (+ its history CSV) if present and
# writes the checkpoint back into gpurun_out/ (copy it to ckpt/ before the next segment).
# Usage (under gpurun):
#   bash scripts/gpu_longruns.sh foil [cycles] [max-minutes]   |   bash scripts/gpu_longruns.sh cylinder
mkdir -p gpurun_out
case "${1:-foil}" in
  foil)
    [ -f ckpt/f1_M1.npz ] && cp ckpt/f1_M1.npz gpurun_out/f1_M1_ckpt.npz
    python scripts/production_cycles.py --cycles ${2:-3} --max-minutes ${3:-52} --out-prefix gpurun_out/f1_M1 \
        --ckpt gpurun_out/f1_M1_ckpt.npz --history ckpt/f1_M1.csv > gpurun_out/f1_M1.log 2>&1
    tail -c 3000 gpurun_out/f1_M1.log ;;
  cylinder) timeout 1500 python scripts/validate_cylinder.py --nx 1024 --ny 768 --dt 0.01 --steps 8000 --omega-p 1.98 \
          --maxit-p 30000 --out gpurun_out/cylinder_1024x768 > gpurun_out/cyl1024.log 2>&1; tail -c 1500 gpurun_out/cyl1024.log ;;
esac
