"""Trace-CSV fixtures from the REFERENCE (moesim.workload.export_trace / load_trace,
workload.py:14, :145-178) for serving.export_trace / load_trace.

Run only in the build container (needs /root/reference):

    python tests/golden/make_trace.py

Writes tests/golden/trace_arxiv10.csv (the reference's export of the first 10
requests of the configs/qwen_arxiv_*.toml workload, seed 2) and
tests/golden/trace_errors.json (the reference's error text for malformed files).
"""

import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    from moesim.types import ValidationError
    from moesim.workload import LogNormalLengths, WorkloadConfig, export_trace, generate_requests, load_trace

    wl = WorkloadConfig(request_rate_rps=1.3, seed=2, num_requests=10,
                        length_dist=LogNormalLengths(9194, 5754, 231, 104))
    reqs = generate_requests(wl)
    export_trace(reqs, os.path.join(HERE, "trace_arxiv10.csv"))
    bad = {"wrong_fields": "id,arrival_s,input_len,output_len\n0,0.0,10,5\n1,0.5,7\n",
           "not_a_number": "id,arrival_s,input_len,output_len\n0,0.0,10,5\n1,zero,7,3\n"}
    errors = {}
    with tempfile.TemporaryDirectory() as d:
        for name, text in bad.items():
            p = os.path.join(d, name + ".csv")
            with open(p, "w") as f:
                f.write(text)
            try:
                load_trace(p)
                errors[name] = None
            except ValidationError as exc:
                errors[name] = {"text": text, "message": str(exc).replace(p, "<path>")}
    with open(os.path.join(HERE, "trace_errors.json"), "w") as f:
        json.dump(errors, f, indent=1)
    print(len(reqs), "requests;", errors)


if __name__ == "__main__":
    main()
