import json,sys
d=json.load(open(sys.argv[1])); k=d["kernels"]
print(sys.argv[1], d["value"], d["e2e"]["value"], "A %.3f AT %.3f qr %.3f" % (k["spmv_A"]["ms_total"]/k["spmv_A"]["launches"], k["spmv_AT"]["ms_total"]/k["spmv_AT"]["launches"], k["qr_step"]["ms_total"]/k["qr_step"]["launches"]), d["clocks"]["sm_mhz"])
