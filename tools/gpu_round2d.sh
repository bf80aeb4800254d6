# round-2 final GPU pass: tests, smoke, bench lines for every config, ncu launch list + full capture
set -x
TAG=${TAG:-r02d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 300 python bench.py > gpurun_out/${TAG}_bench_b.json 2> gpurun_out/${TAG}_bench_b.err
timeout 600 python bench.py --config C --steps 30 > gpurun_out/${TAG}_bench_c.json 2> gpurun_out/${TAG}_bench_c.err
timeout 900 python bench.py --config D --steps 10 > gpurun_out/${TAG}_bench_d.json 2> gpurun_out/${TAG}_bench_d.err
timeout 600 python bench.py --config E --steps 10 > gpurun_out/${TAG}_bench_e.json 2> gpurun_out/${TAG}_bench_e.err
timeout 300 python bench.py --config R --steps 200 > gpurun_out/${TAG}_bench_r.json 2> gpurun_out/${TAG}_bench_r.err
timeout 300 python bench.py --config M --steps 20 > gpurun_out/${TAG}_bench_m.json 2> gpurun_out/${TAG}_bench_m.err
timeout 300 python bench.py --config O --steps 20 > gpurun_out/${TAG}_bench_o.json 2> gpurun_out/${TAG}_bench_o.err
timeout 600 python bench.py --config L --steps 10 > gpurun_out/${TAG}_bench_l.json 2> gpurun_out/${TAG}_bench_l.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 300 python tools/timeline.py > gpurun_out/${TAG}_timeline.txt 2>&1
K='regex:logits|lg_final|select_k|attn_tma|tma_merge|attn_bf16|norm_k|group_k|topk|diff_k|gather|merge|rethead'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 40 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:logits_tma|attn_tma|select_k|tma_merge" -s 8 -c 4 -o gpurun_out/${TAG}_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/ | grep $TAG
