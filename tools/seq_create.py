import os, sys, torch
sys.path.insert(0, os.getcwd())
import graphgen, paper_2109_09527_b200 as pr
def t(k):
    gen = graphgen.make_config(k)
    s = torch.from_numpy(gen.src).cuda(); tt = torch.from_numpy(gen.dst).cuda()
    st = torch.cuda.current_stream()
    w = pr.Graph(gen.n, s, tt); w.preprocess(); w.close()
    cts = []
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); g = pr.Graph(gen.n, s, tt); b.record(st); torch.cuda.synchronize()
        cts.append(a.elapsed_time(b)); g.preprocess(); g.close()
    print(k, os.environ.get("PRGPU_PACK"), [round(c, 2) for c in cts], flush=True)
    del s, tt; torch.cuda.empty_cache()
for k in [int(a) for a in sys.argv[1:]]: t(k)
