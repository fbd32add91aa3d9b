import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_05345_b200.rasterizer import microbench_red
for rep in range(2):
    print({p: round(microbench_red(p, 1<<28)/1e9,1) for p in range(10)})
