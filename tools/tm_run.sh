for v in tmc2x5 tmc3 tmc3x5; do echo $v; timeout 300 python tools/step_parts.py --lib=tools/libspc_$v.so | grep -E "^A |^LSA"; done
