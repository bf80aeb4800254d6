# A/B of the register-direct attention (needs tools/attn_ldg_experiment.cuh.txt restored as csrc/attn_ldg.cuh + its dispatch in attn.cu; SPC_ATTN_LDG=2|4) against the default path
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 2 4; do
  SPC_ATTN_LDG=$v timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_pipeline.py -q -x 2>&1 | tail -2
done
for v in 0 2 4 0 2 4; do
  echo "LDG=$v"; SPC_ATTN_LDG=$v timeout 300 python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline'])"
done
