"""Loss reproducibility across launches: synthetic weights / inputs come from
process-stable seeds, so two launches must start from identical values.  Prints the
per-step losses of a few training steps (fp32 repr) for comparison across runs."""
import json
import sys

import torch

from paper_2201_12023_b200.runtime import Executor


def main():
    plan = sys.argv[1] if len(sys.argv) > 1 else "plans/gpt13b_block1_n1/plan.json"
    ex = Executor(plan, schedule="1f1b", seed=1234)
    losses = []
    for _ in range(3):
        ex.step()
        losses.append(ex.loss())
    w = ex.runner.wbf16.float()
    print(json.dumps({"losses": [repr(x) for x in losses],
                      "weights_checksum": repr(float(w.double().sum()))}))


if __name__ == "__main__":
    main()
