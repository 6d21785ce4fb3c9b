# wide-kernel staging depth A/B: default (4 ring stages, 2 x 4 KB staging per epilogue warp) vs 3 stages + 5 / 4 staging tiles
python paper_2605_21442_b200/build.py >/dev/null
run() {  # lib cfg
  if [ "$1" = default ]; then unset LCE_LIB_PATH; else export LCE_LIB_PATH=$PWD/ab/liblce_$1.so; fi
  timeout 600 python bench.py --config $2 --path fused --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-split 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$2 $1', round(d['value']), round(d['ms_per_step_median'],3), 'dW', round(k['bwd_dw']['ms_per_step'],2), round(k['bwd_dw']['util_at_clock'],3), 'dH', round(k['bwd_dh']['ms_per_step'],2), round(k['bwd_dh']['util_at_clock'],3), d['clocks']['sm_mhz'])"
  unset LCE_LIB_PATH
}
for rep in 1 2 3; do for v in default w3b5 w3b4; do run $v llama8b; done; done
for v in default w3b5; do run $v llama1b; run $v qwen7b; done
