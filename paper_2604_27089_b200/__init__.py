"""AutoSP (arxiv 2604.27089) Ulysses sequence-parallel hot path, B200-native.

User API (Listing 1):
    import paper_2604_27089_b200 as autosp
    autosp.reg_passes(['auto_sp', 'sp_ac'])
    autosp.dist.init(SP_GROUP_SIZE)
    model = autosp.compile(model)          # or model.compile(backend=autosp.backend())
    loss = model(batch[:, sp_slice]); loss.backward(); opt.step()
"""

from .errors import (CollectiveError, EquivalenceError, ExtensionMissingError, InfeasibleError,
                     SeqcompError, UnsupportedError, ValidationError)

__all__ = ["CollectiveError", "EquivalenceError", "ExtensionMissingError", "InfeasibleError",
           "SeqcompError", "UnsupportedError", "ValidationError"]
