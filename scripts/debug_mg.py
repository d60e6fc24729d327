import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle.rng import chain
from oracle.sampler import sample_micrograph as o_sample, stream_key
from paper_2409_00657_b200.graph import Graph
from paper_2409_00657_b200.sampler import MicrographBuilder
g = np.load('tests/golden/micrographs.npz')
G = Graph.from_host(g['offsets'], g['targets'])
seed = int(g['seed'][0])
roots = g['roots'][:3]
for fo in [(7,), (15, 10)]:
    b = MicrographBuilder(fo, len(roots))
    st = torch.tensor([np.uint64(chain(seed, 1, 2)).view(np.int64)], device='cuda')
    batch = b.build(G, torch.from_numpy(roots).cuda(), st, len(roots))
    torch.cuda.synchronize(); b.check()
    h = batch.to_host()
    print('fo', fo, 'totals', batch.totals.cpu().numpy())
    for k in range(len(fo)+1):
        print(' k', k, 'need_off', h['need_off'][k][:4], 'ids', h['need_ids'][k][:20], 'inl', h['in_layer'][k][:20])
    ms = batch.micrographs(roots)
    for r, m in zip(roots.tolist(), ms):
        w = o_sample(g['offsets'], g['targets'], r, fo, stream_key(seed, 1, 2, r))
        print(' root', r, 'deg', g['offsets'][r+1]-g['offsets'][r])
        print('   got layers', [x.tolist() for x in m.layers])
        print('   want layers', [x.tolist() for x in w.layers])
    ws = b.ws.cpu().numpy()[:b.layout.ws_root_ints]
    print(' ws root0', ws[:80])
