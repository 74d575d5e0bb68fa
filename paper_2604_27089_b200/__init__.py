"""AutoSP (arxiv 2604.27089) Ulysses sequence-parallel hot path, B200-native.

User API (Listing 1):
    import paper_2604_27089_b200 as autosp
    autosp.reg_passes(['auto_sp', 'sp_ac'])
    autosp.dist.init(SP_GROUP_SIZE)
    model = autosp.compile(model)           # model.compile(backend=autosp.backend())
    loss = model(batch[:, sp_slice]); loss.backward()   # grads summed over SP in-graph
    opt.step()
"""

from . import dist
from .auto_sp import positions
from .compiler import backend, compile, reg_passes, registered_passes
from .errors import (CollectiveError, EquivalenceError, ExtensionMissingError, InfeasibleError,
                     SeqcompError, UnsupportedError, ValidationError)
from .sp_ac import AcMode

__all__ = ["dist", "positions", "backend", "compile", "reg_passes", "registered_passes",
           "AcMode", "CollectiveError", "EquivalenceError", "ExtensionMissingError",
           "InfeasibleError", "SeqcompError", "UnsupportedError", "ValidationError"]
