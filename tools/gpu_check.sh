#!/bin/bash
# GPU suite + default bench + unskew A/B (TMA vs register-staged) at configs 2/4 + write bandwidth.
O=gpurun_out/${1:-chk}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -n 2 $O/pytest.log
timeout 300 python tools/write_bw.py > $O/write_bw.json 2>&1; cat $O/write_bw.json
timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print('bench', round(d['ms_per_step'],3), d['clocks'], {k: round(v,3) for k,v in d['phase_ms_per_step'].items()})"
SKIP_TESTS=1 bash tools/unskew_ab2.sh ${1:-chk}/ab
