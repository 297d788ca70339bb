import numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2410_01626_b200 as cph
from oracle import pairlist as OPL
from synthetic.systems import make_system
s = make_system(2)
ctx = cph.cph_create(s, [4.0], [1])
got = ctx.cph_get_pairlist(0)
ref = OPL.canonical_pairs(s.pos, s.box, 1.1, s.excl)
g = set(map(tuple, got.tolist())); r = set(map(tuple, ref.tolist()))
print('got', len(g), 'ref', len(r), 'missing', len(r - g), 'extra', len(g - r))
x = s.pos.astype(np.float64)
for (i, j) in list(r - g)[:8] + list(g - r)[:8]:
    d = x[j] - x[i]; d -= s.box * np.round(d / s.box)
    print(i, j, np.sqrt((d * d).sum()), x[i], x[j])
