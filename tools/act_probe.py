"""Which cluster-kernel instantiation a config's bonds get and how many clusters
it keeps resident (dev library, TTP_DEBUG_ACT): config 5 (16448 x 64 blocks)
reports act_tp=74 act_lat=74, i.e. the 512-thread shape at one CTA per SM,
so a chunk of 74 options fills the machine exactly once per kernel."""
import os, sys
os.environ["TTP_DEV_LIBRARY"]="1"; os.environ["TTP_DEBUG_ACT"]="1"
sys.path.insert(0,".")
import paper_2203_02804_b200 as P
from paper_2203_02804_b200 import configs
sp=configs.CONFIGS[5]
cfg=P.CrossConfig(bond_dim=sp.bond_dim, seed=sp.cross_seed, max_sweeps=1)
shape=(sp.grid.points_per_axis,)*sp.d
P.tt_cross_batch([P.PhiGridOracle(configs.make_model(5,i), sp.grid) for i in range(2)], shape, cfg, with_reports=False)
