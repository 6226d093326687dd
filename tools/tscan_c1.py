import sys, statistics, torch
sys.path.insert(0, '.')
import paper_2307_11339_b200 as hs
for T in (1, 16, 64, 256):
    spec = hs.CONFIGS['c1'].with_(seq=T)
    ex = hs.RNNExecutor(spec, hs.init_weights(spec)); x = hs.make_input(spec).cuda(); outs = ex.alloc_outputs()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(60):
        e0.record(); ex.forward(x, out=outs); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    print(T, statistics.median(ts[10:]))
