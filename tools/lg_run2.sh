for v in nomath nc4 b1 b4; do echo $v; python tools/lg_graph.py --lib=tools/libspc_$v.so; done
python tools/lg_graph.py
head -30 tools/tmatile.cu | grep -i -E "usage|nvcc" 
