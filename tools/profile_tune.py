import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'bench_tune.py')).read().split('out = {}')[0])
from paper_2312_05385_b200 import _native as nat
for _ in range(3): tune(recs, ramps, TunerParams(), prof, evaluator=ev, device_loop=True)
nat.profile_read(); nat.profile_enable(True)
t0=time.perf_counter()
for _ in range(10): tune(recs, ramps, TunerParams(), prof, evaluator=ev, device_loop=True)
t1=time.perf_counter()
nat.profile_enable(False)
print(nat.profile_read(), (t1-t0)/10*1e3, 'ms wall per tune')
