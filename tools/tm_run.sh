timeout 300 python tools/step_parts.py | grep -E "^A |^LSA"
for v in pf2 pf6 pf8; do echo $v; timeout 300 python tools/step_parts.py --lib=tools/libspc_$v.so | grep -E "^A |^LSA"; done
