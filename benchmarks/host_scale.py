"""Host cost of replica 0's scheduler as the closed loop grows with N (CPU only).

PoolRuntime over host-only workers whose forward sleeps for a config-2 step's GPU time
(12.5 ms): the process CPU time per step is the scheduler's work (dispatch, routing,
executor timers, completions) for 256 workflows (N = 1) and for 2 048 (N = 8, 4 + 4
engines). Replica 0 must stay under the GPU's step time for weak scaling to hold.
    python benchmarks/host_scale.py
"""
import sys, time
ROOT = __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, ROOT + '/tests')
from harness import HostWorker
from paper_2510_14126_b200.engine import EngineParams, blocks_for
from paper_2510_14126_b200.runtime import PoolRuntime
from paper_2510_14126_b200.workflow import Nl2Sql

class SlowWorker(HostWorker):
    def forward(self, plan):
        time.sleep(0.0125)  # a config-2 step's GPU time
        return super().forward(plan)

for conc, epp in ((256, (1, 1)), (2048, (4, 4))):
    mb = 2 * 256 if epp != (1, 1) else 256
    p = EngineParams(1000 + mb * 450, 5000.0, 0.02, 0.1, mb)
    n_eng = sum(epp)
    w = SlowWorker(n_eng * blocks_for(p), n_eng * (mb + 4))
    rt = PoolRuntime(w, Nl2Sql(retry_budget=5), p, mode="isolated", engines_per_pool=epp,
                     concurrency=conc)
    rt.fill()
    rt.run_steps(400)
    c = time.process_time(); t = time.perf_counter()
    rt.run_steps(200)
    dc = (time.process_time() - c) / 200; dt = (time.perf_counter() - t) / 200
    print(conc, epp, f"host CPU {dc*1e3:.2f} ms per step, wall {dt*1e3:.2f} ms (forward sleeps 12.5 ms)",
          "completed", rt.stats.completed)
