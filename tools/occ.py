import ctypes, torch
print(torch.cuda.get_device_properties(0))
