import sys; sys.path.insert(0,'.')
from paper_2110_12952_b200 import *
T=builtin_descriptor("sierpinski-triangle")
s=Simulation(T,6,Backend.GpuBoundingBox); s.seed_random(3,0.5); s.step(conway_rule()); print("ok", s.state_hash())
