import sys, time, torch
sys.path.insert(0, '/root/repo')
import synth
from paper_1207_1773_b200 import Solver, colmajor
n = int(sys.argv[1])
s = Solver(0, nb=64)
A0 = colmajor(synth.rand_hermitian(n, 0), torch.device('cuda:0'))
for P in (1, 2, 4, 8):
    A = A0.clone(); s.he2hb_sim(A, P); torch.cuda.synchronize()
    t = time.perf_counter(); A = A0.clone(); s.he2hb_sim(A, P); torch.cuda.synchronize()
    print(f"he2hb_sim n={n} P={P} (all virtual ranks on one GPU, sequential): {(time.perf_counter()-t)*1e3:.1f} ms")
