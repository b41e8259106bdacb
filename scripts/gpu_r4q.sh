#!/bin/bash
# least-squares degree of the band guess per level (dt = T/128, T/256, T/512)
cd "$(dirname "$0")/.."
for lvl in 1 2 3; do
  steps=$((512 << (lvl - 1)))
  for d in 6 5 4; do
    echo -n "level=$lvl steps=$steps lsdeg=$d  "
    TILE_AB_LEVEL=$lvl MLMCP_BAND_LSDEG=$d timeout 300 python scripts/tile_ab.py 2 112 $steps band 2>&1 | grep '"mode"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['call_ms'], d['its_per_step'])"
  done
done
