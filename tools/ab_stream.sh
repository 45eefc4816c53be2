# A/B of two liblb builds on the hot-plan merge-path step (C3, C4), alternating, 3 rounds each
for i in 1 2 3; do for lib in "$@"; do
  LB_LIB_PATH=$lib python tools/sweep_hot.py c3,c4 16384 16 1016 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'slots' in d: print('$lib', d['config'], d['GNZ/s'], d['GNZ/s_cached'])"
done; done
