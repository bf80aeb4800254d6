# one GPU call: tests, bench lines for configs B/C/E, ncu launch list + full capture (tools only)
set -x
TAG=${TAG:-r01g}
python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
python bench.py > gpurun_out/${TAG}_bench_b.json 2> gpurun_out/${TAG}_bench_b.err
python bench.py --config C --steps 30 > gpurun_out/${TAG}_bench_c.json 2> gpurun_out/${TAG}_bench_c.err
python bench.py --config E --steps 10 > gpurun_out/${TAG}_bench_e.json 2> gpurun_out/${TAG}_bench_e.err
K='regex:logits|lg_final|select_k|attn_bf16|norm_k|group_k|topk|diff_k|gather|merge'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:logits_kernel|attn_bf16|select_k" -s 6 -c 3 -o gpurun_out/${TAG}_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/
