"""Live Philox4x32-10 block-rate probe (development tool): gsb_philox_bench."""
import sys; sys.path.insert(0,'.')
import torch
from paper_2505_18508_b200 import _lib
L=_lib.lib()
dev=torch.device('cuda',0); sink=torch.zeros(256,dtype=torch.int32,device=dev)
s=torch.cuda.current_stream().cuda_stream
nthr=torch.cuda.get_device_properties(0).multi_processor_count*8*256
for bpt in [64,4096,4096,8192]:
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); _lib.check(L.gsb_philox_bench(bpt, sink.data_ptr(), s)); e1.record(); torch.cuda.synchronize()
    print(bpt, nthr*bpt/(e0.elapsed_time(e1)/1e3)/1e9, "Gblock/s")
