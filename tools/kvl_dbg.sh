for args in "0 37 tiny" "1 37 tiny" "0 200 tiny" "0 300 0" "2 300 0" "2 8192 3"; do timeout 60 python tools/kvl_dbg.py $args 2>&1 | grep -E "^ok|Error|error" | head -2; done
DCOPF_DEBUG_MODE=1 timeout 60 python tools/kvl_dbg.py 1 37 tiny 2>&1 | grep -E "^ok|Error" | head -2
DCOPF_DEBUG_MODE=2 timeout 60 python tools/kvl_dbg.py 1 37 tiny 2>&1 | grep -E "^ok|Error" | head -2
