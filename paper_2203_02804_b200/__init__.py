"""B200-native TT-Fourier multi-asset option pricer (arXiv 2203.02804 hot path).

Drop-in for the reference package's pricing API (``ttpricer``): same names,
signatures and exceptions for the hot path -- ``price_fourier_tt``,
``tt_cross``, ``tt_inner``, ``maxvol``, ``tt_evaluate_many``,
``tt_rand_sample_diff``, ``price_fourier_dense`` -- with every numerical step
executed by hand-written sm_100a kernels behind the C ABI in
``include/ttpricer_b200.h``.  Batched variants (``*_batch``) price many
independent options per call.
"""

__version__ = "0.1.0"

from .errors import (
    CapacityError,
    DeviceError,
    MaxvolIterationError,
    NumericsError,
    OracleBudgetError,
    ResidueError,
    SingularMatrixError,
    StripConditionError,
)
from .market import MarketModel, black_scholes_price, corr_matrix_plus
from .oracles import (
    DeviceOracle,
    OracleBatch,
    PayoffGridOracle,
    PhiGridOracle,
    SeparableOracle,
    TableOracle,
    TTOracle,
)
from .tensor_train import (
    TensorTrain,
    sample_indices,
    tt_evaluate,
    tt_evaluate_many,
    tt_inner,
    tt_inner_batch,
    tt_load_json,
    tt_rand_sample_diff,
    tt_save_json,
)
from .cross import CrossConfig, CrossReport, column_basis, maxvol, tt_cross, tt_cross_batch
from .pricers import (
    DENSE_TERM_CAP,
    GridSpec,
    PricingResult,
    grid_admissible,
    payoff_grid_oracle,
    phi_grid_oracle,
    price_fourier_dense,
    price_fourier_dense_batch,
    price_fourier_tt,
    price_fourier_tt_batch,
    price_strike_ladder,
    table1_hyperparams,
)
from .montecarlo import price_monte_carlo, price_monte_carlo_batch
from .experiments import ExperimentConfig, run_bond_dim_sweep, run_strike_sweep, run_table1

__all__ = [name for name in dir() if not name.startswith("_")]
