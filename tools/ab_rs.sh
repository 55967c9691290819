# A/B of the options held during the rank-stream wavefront (PINTLAB_RANK_STREAM_OPTS); "-" = built-in
for o in "$@"; do
  if [ "$o" = "-" ]; then unset PINTLAB_RANK_STREAM_OPTS; else export PINTLAB_RANK_STREAM_OPTS="$o"; fi
  timeout 300 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$o', round(d['value'],3), round(d['ms_per_step'],1), 'e2e', round(d['e2e']['value'],3))"
done
