# the whole GPU suite on liblce_debug.so (every device spin wait traps after 2 s): no wait anywhere comes near it
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
LCE_LIB_PATH=$PWD/paper_2605_21442_b200/liblce_debug.so timeout 2700 python -m pytest tests -m gpu -q 2>&1 | tail -4
