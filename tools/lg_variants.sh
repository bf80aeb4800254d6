# LOGITS tile-height / warp-count variants: parity of the score + select tests, config-B step time
for v in "" "SPC_LG_RPT=2 SPC_LG_WARPS=10" "SPC_LG_RPT=2 SPC_LG_WARPS=8" "SPC_LG_RPT=2 SPC_LG_WARPS=11" "SPC_LG_RPT=4 SPC_LG_WARPS=6"; do
  echo "== [$v]"
  python -c "
import sys; sys.path.insert(0, '.')
from paper_2512_00722_b200 import build
build.build(force=True, defines=[d for d in '$v'.split() if d])" || continue
  timeout 600 python -m pytest tests/test_gpu_score.py tests/test_gpu_select.py -q -x 2>&1 | tail -1
  for r in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1000,2), 'us', round(d['value']))"; done
  timeout 300 python bench.py --no-cpu-baseline --config E --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('E', round(d['ms_per_step']*1000,2), 'us')"
done
