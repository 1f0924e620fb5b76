# Tile size at C4 scale: default (8192) vs 4096 / 16384, 1-GPU C4 bench and the N-rank proxy.
cd $GRAFT_REPO_ROOT
for r in 1 2; do for t in default 4096 16384; do
  if [ $t = default ]; then unset FCM_TILE_EXPERIMENT; else export FCM_TILE_EXPERIMENT=$t; fi
  timeout 600 python bench.py --config C4 --no-cpu-baseline --steps 10 > gpurun_out/tile_${t}_$r.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tile_${t}_$r.json')); print('tile $t run$r C4', round(d['value']/1e9,2), 'G')"
  timeout 600 python tools/rank_proxy.py 2>&1 | grep -E "^ [1248] " | sed "s/^/tile $t run$r /"
done; done
