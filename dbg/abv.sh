# interleaved variants: bash dbg/abv.sh CONFIGS RUNS_REGEX ROUNDS "label:ENV=.. ENV2=.." ...   (label old -> dbg/old lib)
CONFIGS=$1; PAT=$2; ROUNDS=$3; shift 3
for i in $(seq $ROUNDS); do for spec in "$@"; do
 label=${spec%%:*}; envs=${spec#*:}
 if [ "$label" = old ]; then lib="FASTCONV_LIB=$PWD/dbg/old/libfastconv.so"; else lib=""; fi
 env $lib $envs timeout 200 python tools/bench_configs.py --configs $CONFIGS --steps 50 --tag abv > /dev/null 2>&1
 python - "$label" "$PAT" <<'PY'
import json, re, sys
v, pat = sys.argv[1], sys.argv[2]
d = json.load(open('profiles/abv_configs.json'))
print(v.ljust(6), ' '.join('%s/%s:%.4f[%s]' % (c[:5], k.replace('winograd', 'W').replace('regular_fft', 'R').replace('gauss_fft', 'G'),
      r['ms'], ','.join('%.3f' % x for x in r['stage_ms'])) for c, vv in d['configs'].items() for k, r in vv['runs'].items()
      if re.search(pat, k)))
PY
done; done
