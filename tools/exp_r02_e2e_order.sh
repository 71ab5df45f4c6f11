# e2e (sb_execute_async, two contexts ping-ponging): kernel phases ordered across the contexts
# (sb_context_set_kernel_order) vs free-running, back to back on one box
set -u
python -m pytest tests/test_gpu_conv.py -q -k pingpong > gpurun_out/order_tests.log 2>&1; echo EXIT $? >> gpurun_out/order_tests.log
for rep in 1 2; do
for v in ordered unordered; do
  if [ $v = unordered ]; then export SB_E2E_UNORDERED=1; else unset SB_E2E_UNORDERED; fi
  python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('$v', 'device', d['ms_per_step'], 'ms', d['value'], 'e2e', e['value'], e.get('kernel_order'), 'ms/step', round(d['algorithmic_ops_per_step'] if 'algorithmic_ops_per_step' in d else 0))" >> gpurun_out/order_ab.log 2>&1
done; done
unset SB_E2E_UNORDERED
