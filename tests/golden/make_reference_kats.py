"""Writes tests/golden/reference_kats.json: the known-answer vectors of the
reference's own doctest files (/root/reference/proj/tests/*.cpp), transcribed
with their file:line so the fixture can be re-checked against the source.

The reference cannot be built here (Eigen3 / doctest absent), so
these in-source constants are its golden vectors; tests/test_golden.py runs
them against the oracle and (GPU) the device library.

  python tests/golden/make_reference_kats.py
"""
import json
from pathlib import Path

KATS = {
    "split_in_order": [  # test_packseq.cpp:14-35
        {"src": "test_packseq.cpp:14-35", "lengths": [2, 1, 3, 6, 4], "B": 2, "order": [0, 1, 2, 3, 4],
         "group_lengths": [[2, 1, 3, 2], [4, 4]], "group_skips": [[0, 0, 0, 0], [2, 0]],
         "group_steps": [8, 8]},
    ],
    "pack_batch_sizes": [  # test_packseq.cpp:60-80
        {"src": "test_packseq.cpp:60-70", "lengths": [3, 2, 1], "batch_sizes": [3, 2, 1]},
        {"src": "test_packseq.cpp:72-76", "lengths": [5], "batch_sizes": [1, 1, 1, 1, 1]},
        {"src": "test_packseq.cpp:77-80", "lengths": [4, 4], "batch_sizes": [2, 2, 2, 2]},
    ],
    "gae": [  # test_learner.cpp:72-97
        {"src": "test_learner.cpp:72-81", "lengths": [3], "gamma": 1.0, "lambda": 1.0,
         "reward": [1.0, 0.0, 0.0], "value": [0.0, 0.0, 0.0], "done": [0, 0, 1], "bootstrap_valid": 0,
         "advantage": [1.0, 0.0, 0.0]},
        {"src": "test_learner.cpp:90-97", "lengths": [2, 2], "gamma": 0.99, "lambda": 0.95,
         "reward": [0.0, 3.0, 0.0, 0.0], "value": [0.0, 1.0, 0.0, 0.0], "done": None,
         "bootstrap_valid": None, "check_index": 1, "check_advantage": 2.0},
    ],
    "estimate_time": [  # test_distributed.cpp:61-79
        {"src": "test_distributed.cpp:61-70", "tau": [0.5, 0.5, 0.5, 0.5], "max_steps": 40,
         "steps": [0, 1, 4, 5, 11], "time": [0.0, 0.5, 0.5, 1.0, 1.5]},
        {"src": "test_distributed.cpp:72-79", "tau": [1.0, 2.0], "max_steps": 10,
         "steps": [1, 2, 3], "time": [1.0, 2.0, 2.0]},
    ],
    "optimal_preempt_steps": [  # test_distributed.cpp:104-110
        {"src": "test_distributed.cpp:104-110", "tau": [1.0, 1.0], "learn_time": 100.0, "max_steps": 16,
         "s_star": 16},
    ],
    "sequence_lengths": [  # test_rollout.cpp:116-131 (T=3, N=2, Variable)
        {"src": "test_rollout.cpp:116-131", "T": 3, "N": 2,
         "records": [[0, 0, 0, 0], [0, 0, 1, 1], [0, 1, 0, 0], [1, 0, 0, 0], [1, 0, 1, 0], [1, 0, 2, 0]],
         "record_fields": ["env", "episode", "t", "done"], "seq_lengths": [2, 1, 3]},
    ],
}

if __name__ == "__main__":
    out = Path(__file__).with_name("reference_kats.json")
    out.write_text(json.dumps(KATS, indent=1) + "\n")
    print(out)
