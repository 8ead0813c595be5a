# quick GPU check: bench (no CPU legs) + optional pytest selection
#   gpurun -- 'bash tools/gpu_quick.sh TAG [pytest -k expr]'
TAG=${1:-q}
timeout 900 python bench.py --no-cpu-baseline --no-cold > gpurun_out/${TAG}_bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/${TAG}_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['config']
print('ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'K', c['K'], 'B', c['B'], 'U', c['U'], 'regs', c['regs'], 'w', c['w_plan_fp64_ops_per_step'], 'rel_err', d.get('rel_err'), 'plain_ms', d.get('plain_sweep',{}).get('ms_per_step'), 'plain_frac', d.get('plain_sweep',{}).get('roofline',{}).get('frac'))"
if [ -n "$2" ]; then timeout 2400 python -m pytest tests -m gpu -q -x $2 > gpurun_out/${TAG}_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/${TAG}_tests.log; fi
