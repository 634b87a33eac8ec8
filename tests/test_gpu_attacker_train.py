"""LSTM attacker training on a B200: the dataset comes
from the device trace pipeline, training lowers the loss and the
validation LER below an untrained predictor's, and the exported predictor
decodes through tobf_lstm_ctc bit-exactly against the CPU oracle."""

import numpy as np
import pytest

from oracle import fitness_ref as FR
from paper_2107_09789_b200 import attacker
from paper_2107_09789_b200.attacker_train import (ArchGenConfig, TrainParams, build_dataset, dataset_ler,
                                                  train_predictor)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2107_09789_b200.engine import device
    return device(0)


def test_train_and_export(ctx):
    ds = build_dataset(160, ArchGenConfig(seed=1))
    assert len(ds.labels) == 160 and ds.feats.shape[1] == 9 and ds.offsets[-1] == len(ds.feats)
    pred, hist = train_predictor(ds, TrainParams(hidden=64, epochs=25, seed=0))
    assert hist["train"][-1] < 0.5 * hist["train"][0]
    val = hist["val_idx"]
    untrained = attacker.init_predictor(64, seed=5)
    assert dataset_ler(ds, pred, val) < dataset_ler(ds, untrained, val)
    # exported weights are bf16-representable and decode bit-exactly like the oracle
    for w in pred.weights().values():
        assert np.array_equal(w, attacker._bf16_round(w))
    for i in val[:8]:
        lo, hi = ds.offsets[i], ds.offsets[i + 1]
        import torch
        f = torch.from_numpy(np.ascontiguousarray(ds.feats[lo:hi])).to(ctx.device)
        offs = torch.tensor([0, hi - lo], dtype=torch.int32, device=ctx.device)
        toks, ntok = attacker.decode(f, offs, 1, int(hi - lo), pred)
        got = list(toks.cpu().numpy()[0, :int(ntok.cpu()[0])])
        assert got == FR.lstm_ctc(ds.feats[lo:hi], 9, pred.weights())
