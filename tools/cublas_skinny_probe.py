import torch, time
A=torch.randn(5000,10000,dtype=torch.float64,device="cuda")
Q=torch.randn(10000,133,dtype=torch.float64,device="cuda")
Z=torch.randn(5000,133,dtype=torch.float64,device="cuda")
for f,name in [(lambda: A@Q,"AQ"),(lambda: A.t()@Z,"AtZ")]:
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/10
    print(name, "%.1f us"%(ms*1e3), "%.1f TF"%(2*5000*10000*133/ms/1e9))
