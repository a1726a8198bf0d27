import sys; sys.path.insert(0,'.')
import torch, paper_2106_13465_b200 as P
s=torch.cuda.Stream(); torch.cuda.set_stream(s)
g=P.GpuGrid(256,256,1/256,1/256,P.GasModel(),'transmit',device=0); g.set_stream(s.cuda_stream)
g.init_case('sod_x',0); g.run_async(10); g.sync()
g.reset_counters(); g.set_timing(True)
for k in range(3):
    g.init_case('sod_x',0); g.run_async(10)
g.sync(); print(g.kernel_times())
