"""Dev helper: compare one golden case's all-path outputs GPU vs reference fixture."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1505_01466_b200 as pb
from tests import golden_cases
cases, arrays = golden_cases.load()
name = sys.argv[1]
case = [c for c in cases if c['name'] == name][0]
spec, sch, fb, llr = golden_cases.build_case(case)
exp = golden_cases.expected(case, arrays)
dec = pb.ListDecoder(sch, case['L'], mode='int8' if case['int8'] else 'f32')
cw, pm, ok, pu = dec.decode_paths_batch(llr)
print('ops tail', [(o.kind.value, o.size, o.side) for o in sch.ops[-6:]])
for f in range(len(pu)):
    P = pu[f]
    bad = [t for t in range(P) if not np.array_equal(cw[f, t], exp['path_cw'][f, t])]
    if bad or not np.array_equal(pm[f, :P], exp['path_pm'][f, :P]):
        print('frame', f, 'P', P, 'bad rows', bad)
        print(' pm got', pm[f, :P]); print(' pm exp', exp['path_pm'][f, :P])
        for t in bad[:2]:
            d = np.flatnonzero(cw[f, t] != exp['path_cw'][f, t]); print('  row', t, 'diff at', d)
        break
