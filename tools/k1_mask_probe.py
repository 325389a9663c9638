import sys; sys.path.insert(0,'.')
from paper_2602_20826_b200 import _lib
c=_lib.Corpus(1000000, seed=1, gpu=True)
b=c.batch()
for name,mask in [("all",0x1F),("front_only(no proposed)",0x1E),("proposed_only",0x01),("greedy_only",0x02)]:
    s=_lib.Session(b,148,mask=mask)
    for _ in range(3): s.run()
    t=sorted(s.run() for _ in range(5))
    print(name, t[2])
    s.close()
print("gen_ms", c.gen_ms)
