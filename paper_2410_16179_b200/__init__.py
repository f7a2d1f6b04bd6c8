"""B200 (sm_100a) implementation of MagicPIG's decode-time hot path
(LSH importance-sampled decode attention, arXiv 2410.16179).

The product is the C-ABI library ``libmagicpig.so`` (include/magicpig.h), built
in-tree by ``build.py``; ``binding`` marshals torch tensors to it and ``index``
sequences build/decode (and the sharded variants over torch.distributed).
"""
from . import binding
from .binding import make_config, MagicPIGError
from .index import DecodeSession, MagicPIG, session

__all__ = ["binding", "make_config", "MagicPIG", "MagicPIGError", "DecodeSession", "session"]
