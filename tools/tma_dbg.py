import sys, torch
sys.path.insert(0, '.')
import paper_2410_14117_b200 as uuv
for n, A in ((1 << 20, 'bluerov2'), (200000, 'bluerov2')):
    veh = uuv.bluerov2_params()
    cfg = uuv.engine_config_dict(veh, uuv.TaskSpec(), n, 0, device=0)
    cfg["device"]["pair"] = "on"
    g = uuv.B200EnvBatch(cfg)
    print(n, g.info["tma_pipelined"], g.info["step_kernel_registers"], flush=True)
    act = g.bench_actions_tensor()
    try:
        g.step_tensors(act)
        torch.cuda.synchronize()
        print("ok", flush=True)
    except Exception as e:
        print("ERR", repr(e)[:400], flush=True)
        break
