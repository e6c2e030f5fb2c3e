import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_1812_01307_b200 import solvers, blockops, spectral
d = bench.make_problem()
op = blockops.BlockOperator(d.matrix, blockops.make_partition(*d.shape, 8, 8))
cfg = solvers.SolverConfig(mu=0.0487, lam=0.0, epochs=10**9, monitor_decrease=False)
st = solvers.init_bsgd_state(op, d.y, cfg)
hx = np.zeros(d.shape[1]); hr = np.asarray(d.y).copy()
def step(tm):
    global hx, hr
    t0=time.perf_counter(); st.x = hx; t1=time.perf_counter(); st.r_vec = hr; t2=time.perf_counter()
    solvers.bsgd_tv_iteration(st, op, d.y, cfg); torch.cuda.synchronize(); t3=time.perf_counter()
    hx = st.x; t4=time.perf_counter(); hr = st.r_vec; t5=time.perf_counter()
    tm.append((t1-t0,t2-t1,t3-t2,t4-t3,t5-t4))
tm=[]
for _ in range(5): step(tm)
tm=[]
for _ in range(20): step(tm)
a=np.array(tm)*1e3
print("set_x set_r iter get_x get_r (ms):", np.round(a.mean(0),3), "total", round(a.sum(1).mean(),3))
import cProfile, pstats
pr=cProfile.Profile(); pr.enable()
for _ in range(10): step([])
pr.disable(); pstats.Stats(pr).sort_stats('tottime').print_stats(12)
