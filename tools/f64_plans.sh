# fp64 router: device time of every (tile height, cluster size) plan at decode sizes
python -m paper_2511_11505_b200.build > /dev/null
P="4,1;4,2;4,4;4,8;2,1;2,2;2,4;2,8;1,1;1,2;1,4;1,8"
FSC_ROUTER_F64=1 FSC_PLANS="$P" python tools/router_time.py qwen3:64 qwen3:256 qwen3:512 qwen3:1024 scout:64 scout:512 dsv2lite:128 dsv2lite:512 dsv2lite:1024 2>&1 | grep -E "router|Error"
FSC_ROUTER_F64=0 python tools/router_time.py qwen3:64 qwen3:256 qwen3:512 qwen3:1024 scout:64 scout:512 dsv2lite:128 dsv2lite:512 dsv2lite:1024 2>&1 | grep -E "router|Error"
