#!/bin/bash
# usage (on the GPU box): tools/variants.sh file.cu 'sed-expr-1' 'sed-expr-2' ...
# builds libchr.so once per variant (the unmodified source first) and prints
# the bench step time + per-kernel times; restores the source at the end.
F=paper_2408_05462_b200/csrc/$1; shift
cp $F /tmp/variant_orig.cu
run() {
  make -C paper_2408_05462_b200/csrc -j16 >/dev/null 2>&1 || { echo "build failed"; return; }
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('  step %.3f ms  e2e %.2f  ' % (d['ms_per_step'], d['e2e']['ms_per_step']) + ' '.join('%s=%.3f' % (k, v['avg_ms']) for k, v in list(d['kernels'].items())[:6]))"
}
echo "base"; run
for e in "$@"; do
  cp /tmp/variant_orig.cu $F
  sed -i "$e" $F
  echo "variant: $e"; run
done
cp /tmp/variant_orig.cu $F
make -C paper_2408_05462_b200/csrc -j16 >/dev/null 2>&1
