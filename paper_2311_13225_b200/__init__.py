"""B200-native sample-based GNN training hot path (NeutronOrch, arXiv 2311.13225).

Drop-in for the reference package ``hetgnn`` (its __init__.py:5-24 surface) on
the hot path: sampler, layer math, embedding store, hotness, training driver.
All compute runs in the sm_100a library ``libhg_gnn.so`` (C ABI in
include/hg_gnn.h); imports are lazy so that the data-side helpers (datagen,
graph, runplan, seeds) work without a GPU.
"""

__version__ = "0.1.0"

_LAZY = {
    "Block": "sampler", "Fanouts": "sampler", "SampledBlockStack": "sampler", "SamplerError": "sampler",
    "sample_khop": "sampler", "sample_khop_skip_hot": "sampler", "sample_one_hop_hot": "sampler",
    "ModelParams": "gnnmath", "init_params": "gnnmath", "loss_and_grad": "gnnmath", "sgd_step": "gnnmath",
    "HotnessTable": "hotness", "HotSetPartition": "hotness", "estimate_hotness": "hotness",
    "partition_hot": "hotness", "select_hot": "hotness",
    "EmbeddingStore": "store", "StalenessViolation": "store", "StoreContractError": "store",
    "ConfigError": "orchestrator", "EpochReport": "orchestrator", "TrainConfig": "orchestrator",
    "run_training": "orchestrator",
    "Graph": "graph", "VertexData": "graph",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
