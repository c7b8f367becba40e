# A/B of the in-tree library against dbg/old/libfastconv.so, interleaved:
#   bash dbg/ab.sh CONFIGS RUNS_REGEX [ROUNDS]
CONFIGS=$1; PAT=$2; ROUNDS=${3:-3}
for i in $(seq $ROUNDS); do for v in old new; do
 if [ $v = old ]; then export FASTCONV_LIB=$PWD/dbg/old/libfastconv.so; else unset FASTCONV_LIB; fi
 timeout 200 python tools/bench_configs.py --configs $CONFIGS --steps 50 --tag ab_$v > /dev/null 2>&1
 python - "$v" "$PAT" <<'PY'
import json, re, sys
v, pat = sys.argv[1], sys.argv[2]
d = json.load(open('profiles/ab_%s_configs.json' % v))
print(v, ' '.join('%s/%s:%.4f[%s]' % (c[:5], k.replace('winograd', 'W').replace('regular_fft', 'R').replace('gauss_fft', 'G'),
      r['ms'], ','.join('%.4f' % x for x in r['stage_ms'])) for c, vv in d['configs'].items() for k, r in vv['runs'].items()
      if re.search(pat, k)))
PY
done; done
