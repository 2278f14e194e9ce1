"""Kernel-variant coverage: re-run the GPU parity corpus with engine switches
that route every row through the alternative kernels (e.g. the CTA-per-row
chain kernels of chains.cu, normally used only for rows >= 1024 cells), so
each variant is held to the same bit-exact bar against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [{"PC_EXEC_MODE": "1"}, {"PC_EXEC_MODE": "2"}, {"PC_BIG_CHAIN_CELLS": "1"},
                                 {"PC_GBC": "1"}, {"PC_GBC": "0"}, {"PC_GBC": "2"},
                                 {"PC_GBC": "2", "PC_GBC_SMEM_ANY": "1"},
                                 {"PC_EXEC_MODE": "1", "PC_LAZY_COMPACT": "1"}, {"PC_LAG_ROWS": "0"},
                                 {"PC_LAG_ROWS": "1000000"}, {"PC_PIPES": "1"},
                                 {"PC_DENSE_LIVE": "0", "PC_DENSE_V3": "0", "PC_DENSE_V2": "0"},
                                 {"PC_DENSE_V3": "0"}, {"PC_DENSE_TM": "8"},
                                 {"PC_DENSE_TM": "-1"}, {"PC_LIVE_CELLS": "0"}, {"PC_GBC_TILE": "1"},
                                 {"PC_SPLIT_CHAINS": "0"}, {"PC_CHAIN_SCAN": "1"}, {"PC_GBC_FLAT": "0"},
                                 {"PC_RELU_LIST": "0"}, {"PC_PREDICT": "0"}, {"PC_NUMERIC_MODE": "0", "PC_PIPES": "1"},
                                     {"PC_PREDICT": "2"}, {"PC_PRED_DEVICE": "0"}, {"PC_PRED_FUSED": "0"}, {"PC_FWD_STAGED": "0"}, {"PC_MARGIN_PIPE_MIN": "1000000"}, {"PC_PIPES": "3"}, {"PC_FORCE_CHECKED": "1"}],
                         ids=["host_schedule", "graph_schedule", "big_chains", "gbc_tiled", "gbc_legacy",
                              "gbc_smem", "gbc_smem_everywhere", "lazy_compaction", "eager_compaction",
                              "lagged_compaction", "one_pipeline", "dense_all_columns_v1", "dense_ballot_v2", "dense_tm8",
                              "dense_wave_model", "conv_all_cells", "conv_channel_tile", "chains_in_cta",
                              "chains_cta_scan", "conv_live_warp", "relu_chain_scan", "exact_compaction",
                              "one_pipeline_predicted", "predicted_from_exact_constants",
                                  "predicted_compaction_on_host", "predicted_offer_unfused",
                                  "forward_conv_unstaged", "margin_one_pipeline", "three_pipelines", "checked_products_everywhere"])
def test_parity_corpus_under_variant(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(HERE, "test_gpu_parity.py"), "-x", "-q",
                        "-m", "gpu", "-p", "no:cacheprovider"], env=e, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
