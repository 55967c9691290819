# A/B of pl_set_option settings on the default bench (3 steps); args: option strings
for o in "$@"; do
  [ "$o" = "-" ] && o=""
  timeout 300 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline ${o:+--opts $o} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$o', round(d['value'],3), round(d['ms_per_step'],1), d['roofline']['profile_block_shares'].get('mg_mid'))"
done
