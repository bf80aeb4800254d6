python -c "import __graft_entry__ as g; g.build()" > gpurun_out/lg_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_score.py tests/test_gpu_select.py -q -x -m gpu > gpurun_out/lg_tests.log 2>&1; tail -2 gpurun_out/lg_tests.log
python tools/lg_graph.py
python tools/lg_graph.py E
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/lg_bench.json 2> gpurun_out/lg_bench.err
python -c "import json; d=json.load(open('gpurun_out/lg_bench.json')); print(round(d['ms_per_step']*1e3,2), d['config']['phase_us'], d['e2e']['value'])"
python tools/lg_graph.py --lib=tools/libspc_old.so
python tools/lg_graph.py --lib=tools/libspc_old.so E
