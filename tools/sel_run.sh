python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sel_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_select.py tests/test_gpu_pipeline.py -q -x -m gpu > gpurun_out/sel_tests.log 2>&1; tail -3 gpurun_out/sel_tests.log
python tools/sel_graph.py
python tools/sel_graph.py --lib=tools/libspc_old.so
python tools/select_trace.py B 2>&1 | tail -22
