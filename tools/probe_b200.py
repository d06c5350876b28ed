import sys; sys.path.insert(0,'.')
from paper_2209_06800_b200 import probes
for rows, dim in [(232965,16),(232965,64),(2449029,64),(2449029,100),(8_000_000,16)]:
    print('gather', rows, dim, round(probes.gather_gbps(rows, dim, 114_000_000 if dim<=16 else 40_000_000),1), 'GB/s', flush=True)
for nb in [1<<20, 16<<20, 64<<20, 1<<30]:
    print('chase', nb, round(probes.chase_ns(nb),1), 'ns', flush=True)
