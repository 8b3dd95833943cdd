
timeout 400 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 2 -c 1 -o gpurun_out/prof_v7 python -c "
import torch, tools.kbench as k
from paper_2506_22033_b200 import Sampler, SamplingParams
B,V=256,152064
x=(2.0*torch.randn(B,V,device='cuda')).to(torch.bfloat16)
s=Sampler(V,B,max_history=1024,dtype='bf16'); s.set_params(list(range(B)),[SamplingParams(temperature=0.7,top_k=40)]*B)
for i in range(4): s.sample(x,i)
torch.cuda.synchronize()
" > gpurun_out/ncu_v7.log 2>&1
tail -3 gpurun_out/ncu_v7.log
