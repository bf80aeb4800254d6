for v in tmwide tmwide3x4 tmwide6x2; do echo $v; timeout 300 python tools/step_parts.py --lib=tools/libspc_$v.so | grep -E "^A |^LSA"; done
