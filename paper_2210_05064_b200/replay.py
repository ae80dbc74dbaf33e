"""`ver replay` (bench.cpp:373-409) on the GPU learner: load a JSONL rollout
trace (the reference's dump_view format), print its shape and the packed
minibatch shapes, run one PPO update from freshly initialised parameters and
print the update statistics.

  python -m paper_2210_05064_b200.replay trace.jsonl [--seed S] [--minibatches B]
      [--encoder E] [--num-actions A] [--epochs K]
"""
from __future__ import annotations

import argparse
import sys

from . import api as V
from .rng import mix


def run_replay(path: str, seed: int = 1, minibatches: int = 2, encoder: int = 64, num_actions: int = 2,
               epochs: int = 4, out=sys.stdout) -> V.TrainStats:
    view = V.RolloutView.load_jsonl(path)
    h = view.info()
    print(f"trace: {h.size} steps, {h.num_seqs} sequences, N={h.N} T={h.T} deficit={h.deficit}", file=out)
    print("per-env counts: " + " ".join(str(int(c)) for c in view.to_host().per_env_counts), file=out)
    for b, g in enumerate(V.split_minibatches(view, minibatches, seed)):
        pb = V.pack(view, g)
        bs = " ".join(str(int(x)) for x in pb.batch_sizes)
        print(f"mini-batch {b}: {int(sum(pb.batch_sizes))} steps, {len(pb.seqs)} sequences, batch_sizes [{bs}]",
              file=out)
    cfg = V.ModelConfig(obs_dim=h.obs_dim, encoder_dim=encoder, hidden_dim=h.hidden_dim, action_kind=h.action_kind,
                        num_actions=num_actions if h.action_kind == 0 else 0, act_dim=h.act_dim)
    params = V.params_init(cfg, mix(seed, 0x9A9A))
    learner = V.Learner(cfg, params, V.PPOConfig(epochs=epochs, minibatches=minibatches), V.EntropyController(),
                        V.CosineSchedule(), mix(seed, 0xF00D))
    st = learner.update(view)
    print(f"replayed update: loss {st.loss} value_loss {st.value_loss} entropy {st.entropy} "
          f"mean_ratio {st.mean_ratio} clip_fraction {st.clip_fraction}", file=out)
    return st


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("trace")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--minibatches", type=int, default=2)
    ap.add_argument("--encoder", type=int, default=64)
    ap.add_argument("--num-actions", type=int, default=2)
    ap.add_argument("--epochs", type=int, default=4)
    a = ap.parse_args(argv)
    run_replay(a.trace, a.seed, a.minibatches, a.encoder, a.num_actions, a.epochs)
    return 0


if __name__ == "__main__":
    sys.exit(main())
